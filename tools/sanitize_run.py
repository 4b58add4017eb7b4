"""Small run touching every kernel family, for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc
from paper_2006_06890_b200.multi import (CudaPartition, edge_balanced_bounds, local_part,
                                         run_partitions_local)

g = zc.with_uniform_weights(zc.generate_powerlaw(3000, 12.0, 2.0, seed=2))
gu = zc.symmetrized(g)
src = int(zc.pick_sources(g, 1)[0])
for s in ["naive", "merged", "merged-aligned", "packed"]:
    zc.bfs(g, src, s, collect_traffic=s != "packed")
    zc.sssp(g, src, s, collect_traffic=False)
    zc.cc(gu, s, collect_traffic=False)
    zc.pagerank(gu, s, collect_traffic=False, max_iters=5)
dg = zc.DeviceGraph(g)
dg.build_sssp_pairs()
zc.sssp(dg, src, "packed", collect_traffic=False)
b = edge_balanced_bounds(g.offsets, 2)
parts = [CudaPartition(local_part(g, b, k), b, k) for k in range(2)]
run_partitions_local(parts, "bfs", src, "packed")
run_partitions_local(parts, "sssp", src, "merged-aligned", fused=True)
r = zc.generate_rmat(12, 8, seed=1, symmetrize=True)
zc.cc(r, "packed", collect_traffic=False)
print("sanitize run ok")
