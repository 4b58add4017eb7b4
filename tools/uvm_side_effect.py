"""Does running a UVM (managed-memory) traversal slow later zero-copy runs?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc

u = zc.generate_uniform_device(1 << 27, 16, 16, seed=27, weights=(8, 72))
src = int(zc.pick_sources(u.as_csr(), 1, seed=7)[0])
def sssp(tag):
    zc.sssp(u, src, "packed", collect_traffic=False)
    r = zc.sssp(u, src, "packed", collect_traffic=False)
    print(tag, f"sssp packed {r.kernel_ms:.1f} ms", flush=True)
sssp("before")
h = zc.generate_rmat(25, 16, seed=3, placement="hbm")
zc.bfs(h, 1, collect_traffic=False); h.close()
sssp("after-hbm")
m = zc.generate_rmat(25, 16, seed=3, placement="uvm")
m.evict(); zc.bfs(m, 1, collect_traffic=False); m.close()
sssp("after-uvm")
