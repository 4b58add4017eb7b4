"""Is the UVM run cold after evict()?  Times consecutive runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dg = zc.generate_rmat(scale, 16, seed=27, placement="uvm")
src = int(zc.pick_sources(dg.as_csr(), 1, seed=7)[0])
for k in range(3):
    r = zc.bfs(dg, src, collect_traffic=False)
    print("warm" if k else "first", r.kernel_ms, flush=True)
for k in range(2):
    dg.evict()
    r = zc.bfs(dg, src, collect_traffic=False)
    print("after evict", r.kernel_ms, flush=True)
