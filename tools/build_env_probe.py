"""Why the compressed builds run slower inside bench.py than standalone: the
fresh direction-optimizing build (out + in lists) of K27 after the bench's
earlier state is recreated step by step -- (1) nothing, (2) the pinned result
pool (16 x 1 GiB zc_host_alloc buffers held), (3) + bfs_many / bfs results of
the headline, (4) + the OpenMP oracle BFS on the host copy."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
import paper_2006_06890_b200._native as N


def fresh_build(tag):
    dg = zc.generate_rmat(27, 16, seed=27)
    t = time.time()
    dg.build_in_lists()
    dt = time.time() - t
    ph = dg.build_log()
    print(f"[{tag}] fresh out+in build {dt:.2f}s  " +
          " ".join(f"{k}={v:.0f}" for k, v in ph), flush=True)
    return dg


fresh_build("clean").close()
pool = [N.lib().zc_host_alloc(1 << 30) for _ in range(16)]
fresh_build("pinned pool 16 GiB").close()
dg = zc.generate_rmat(27, 16, seed=27)
g = dg.as_csr()
srcs = [int(s) for s in zc.pick_sources(g, 64, seed=7)[:10]]
for r in zc.bfs_many(dg, srcs, "merged-aligned"):
    pass
fresh_build("pool + headline graph + bfs_many").close()
import oracle
t = time.time()
ref = oracle.bfs(g, srcs[0], threads=16)
print(f"oracle bfs {time.time() - t:.1f}s", flush=True)
fresh_build("+ oracle").close()
for p in pool:
    N.lib().zc_host_free(p)
fresh_build("pool freed").close()
