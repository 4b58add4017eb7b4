"""EMGI open at K27: the GPU generator's graph written with store_csr_binary
(the reference's format, csr.py:180-245), then opened by zc_graph_open_emgi
(page-cache reads on 64 MiB chunks in parallel, straight into the pinned
zero-copy buffers) and traversed; wall times of each step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc
path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/k27.emgi"
dg = zc.generate_rmat(27, 16, seed=27)
g = dg.as_csr()
src = int(zc.pick_sources(g, 1, seed=7)[0])
ref = zc.bfs(dg, src, "merged-aligned")
t = time.time()
zc.store_csr_binary(g, path)
print(f"store {time.time() - t:.2f}s ({os.path.getsize(path) / 1e9:.2f} GB)", flush=True)
dg.close()
for rep in range(2):
    t = time.time()
    h = zc.open_emgi(path)
    print(f"open_emgi (page cache) {time.time() - t:.2f}s", flush=True)
    r = zc.bfs(h, src, "merged-aligned")
    assert np.array_equal(r.values, ref.values) and r.traversed_edges == ref.traversed_edges
    h.close()
print("bfs on the opened graph equals the generated one", flush=True)
os.remove(path)
