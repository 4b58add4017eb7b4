"""Config 1 (uniform 2^20 deg 16, the reference's own CPU case): per-call
latency of every strategy -- where per-level host round trips matter."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc

g = zc.generate_uniform(2 ** 20, 16, 16, seed=3)
gw = zc.with_uniform_weights(g)
gu = zc.symmetrized(g)
for placement in ("zerocopy", "hbm"):
    for s in ("merged-aligned", "packed"):
        for algo, graph in (("bfs", g), ("sssp", gw), ("cc", gu)):
            best = None
            for _ in range(5):
                r = zc.cc(graph, s, collect_traffic=False, placement=placement) if algo == "cc" \
                    else getattr(zc, algo)(graph, 0, s, collect_traffic=False, placement=placement)
                if best is None or r.kernel_ms < best.kernel_ms:
                    best = r
            te = best.total_traversed_edges
            print(f"{placement:8s} {algo:4s} {s:15s} iters={best.iterations:3d} kernel={best.kernel_ms:7.3f} ms "
                  f"expand={best.expand_ms:7.3f} ms call={best.total_ms:7.3f} ms "
                  f"GTEPS={te/best.kernel_ms/1e6:7.2f} launches={best.launches}", flush=True)
        zc.release(g); zc.release(gw); zc.release(gu)
