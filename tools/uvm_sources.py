"""Cold-UVM vs zero-copy merged-aligned BFS on the same K27 sources (the
bench's timed sources): per-source device times and ratios."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
srcs = [int(s) for s in zc.pick_sources(zc.generate_rmat(20, 16, seed=27).as_csr(), 1)]  # warm-up
zcg = zc.generate_rmat(27, 16, seed=27)
srcs = [int(s) for s in zc.pick_sources(zcg.as_csr(), 64, seed=7)[3:13]]
zc.bfs(zcg, srcs[0], "merged-aligned", collect_traffic=False)
zt = [zc.bfs(zcg, s, "merged-aligned", collect_traffic=False).kernel_ms for s in srcs]
zcg.close()
u = zc.generate_rmat(27, 16, seed=27, placement="uvm")
ut = []
for rep in range(2):
    for s in srcs:
        zc.evict(u)
        ut.append(zc.bfs(u, s, "merged-aligned", collect_traffic=False).kernel_ms)
for i, s in enumerate(srcs):
    print(f"src {s:10d} zerocopy {zt[i]:7.1f} ms  uvm {ut[i]:7.1f} / {ut[i + len(srcs)]:7.1f} ms  "
          f"ratio {ut[i] / zt[i]:.2f}", flush=True)
print(f"mean ratio {sum(ut[:len(srcs)]) / sum(zt):.3f} (first pass) "
      f"{sum(ut[len(srcs):]) / sum(zt):.3f} (second pass)")
