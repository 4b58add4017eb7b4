import sys, os
sys.path.insert(0, "/root/repo")
import paper_2006_06890_b200 as zc
g = zc.generate_uniform(2**20, 16, 16, seed=3)
dg = zc.device_graph(g)
for _ in range(3):
    r = zc.bfs(dg, 0, "merged-aligned", collect_traffic=False)
print("kernel_ms", r.kernel_ms, "expand_ms", r.expand_ms, "iters", r.iterations, r.traversed_edges)
print("per-level expand ms", [round(x, 3) for x in dg.expand_profile(r.iterations)])
dg.set_tuning("loop=host")
r = zc.bfs(dg, 0, "merged-aligned", collect_traffic=False)
print("host loop kernel_ms", r.kernel_ms)
