"""Small run touching every kernel family, for compute-sanitizer.  Every
handle runs the host-driven level loop (tuning loop=host): the sanitizers'
synccheck / racecheck misreport kernels inside conditional graph nodes
(profiles/r01_sanitizers.txt); `--graph` keeps the default device loop."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc
from paper_2006_06890_b200.multi import (CudaPartition, edge_balanced_bounds, local_part,
                                         run_partitions_local)

GRAPH = "--graph" in sys.argv


def hl(x):
    """x with its device handle on the host-driven level loop."""
    if not GRAPH:
        zc.device_graph(x).set_tuning("loop=host")
    return x


g = hl(zc.with_uniform_weights(zc.generate_powerlaw(3000, 12.0, 2.0, seed=2)))
gu = hl(zc.symmetrized(g))
src = int(zc.pick_sources(g, 1)[0])
for s in ["naive", "merged", "merged-aligned", "packed", "compressed"]:
    zc.bfs(g, src, s, collect_traffic=s not in ("packed", "compressed"))
    zc.sssp(g, src, s, collect_traffic=False)
    zc.cc(gu, s, collect_traffic=False)
    zc.pagerank(gu, s, collect_traffic=False, max_iters=5)
dg = hl(zc.DeviceGraph(g))
dg.build_sssp_pairs()
zc.sssp(dg, src, "packed", collect_traffic=False)
b = edge_balanced_bounds(g.offsets, 2)
parts = [CudaPartition(local_part(g, b, k), b, k) for k in range(2)]
run_partitions_local(parts, "bfs", src, "packed")
run_partitions_local(parts, "sssp", src, "merged-aligned", fused=True)
run_partitions_local(parts, "cc" if not g.directed else "bfs", src, "compressed", fused=True)
run_partitions_local(parts, "sssp", src, "compressed")
# compressed lines: long lists (whole lines) and short lists sharing lines
h = hl(zc.generate_powerlaw(20000, 40.0, 1.8, seed=5))
hs = int(zc.pick_sources(h, 1)[0])
zc.bfs(h, hs, "compressed", collect_traffic=False)
# direction-optimizing: in-list transpose, bottom-up passes, narrowed download,
# pipelined results (widen threads), partitions with bottom-up steps
zc.bfs(h, hs, "direction-optimizing", collect_traffic=False)
hsym = hl(zc.symmetrized(h))
zc.bfs(hsym, hs, "direction-optimizing", collect_traffic=False)
zc.bfs_many(h, [hs, hs + 1], "direction-optimizing")
from paper_2006_06890_b200.multi import generate_rmat_part
rp = [generate_rmat_part(12, 2, k, seed=3) for k in range(2)]
run_partitions_local(rp, "bfs", 1, "direction-optimizing")
r = hl(zc.generate_rmat(12, 8, seed=1, symmetrize=True))
zc.cc(r, "packed", collect_traffic=False)
zc.cc(r, "compressed", collect_traffic=False)
# round 2: work-efficient schedules, symmetric partitions with the fused
# pre-filter and the remote-send count, the default pairs stream
for s in ["merged", "merged-aligned", "packed", "compressed"]:
    zc.cc(r, s, collect_traffic=False, schedule="afforest")
    zc.sssp(g, src, s, collect_traffic=False, schedule="near-far", delta=7)
sp = [generate_rmat_part(12, 2, k, seed=3, symmetrize=True) for k in range(2)]
run_partitions_local(sp, "cc", 0, "merged-aligned", fused=True)
run_partitions_local(sp, "bfs", 1, "merged-aligned", fused=True)
wp = [generate_rmat_part(12, 2, k, seed=3, weights=(1, 9)) for k in range(2)]
run_partitions_local(wp, "sssp", 1, "merged-aligned", fused=True)
# round 2 (late): the radix-sort transposes on unsorted lists (directed
# R-MAT: the fresh out + in build hands the first transpose over as the
# in-lists; then the in-lists of a second handle built after its out-lists;
# sort=segmented for the fallback), the lane-per-list encode, UVM prefetch
q = hl(zc.generate_rmat(13, 16, seed=9))
zc.bfs(q, 1, "direction-optimizing", collect_traffic=False)
q2 = hl(zc.generate_rmat(13, 16, seed=9))
q2.build_compressed()
zc.bfs(q2, 1, "direction-optimizing", collect_traffic=False)
q3 = hl(zc.generate_rmat(13, 16, seed=9))
q3.set_tuning("loop=host,sort=segmented")
zc.bfs(q3, 1, "direction-optimizing", collect_traffic=False)
u = hl(zc.generate_rmat(12, 16, seed=2, placement="uvm"))
u.evict()
u.prefetch()
zc.bfs(u, 1, "merged-aligned", collect_traffic=False)
print("sanitize run ok")
