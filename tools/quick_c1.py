"""Quick timing of config 1 (uniform 2^20 deg 16) on the GPU: each strategy x
placement, plus the link probe.  Development tool, not the bench."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc

print("probe", zc.link_probe(nbytes=1 << 30, iters=5), flush=True)
t = time.time()
g = zc.generate_uniform(2 ** 20, 16, 16, seed=3)
print("gen", time.time() - t, flush=True)
gw = zc.with_uniform_weights(g)
for placement in ("zerocopy", "hbm", "uvm"):
    for s in zc.AccessStrategy:
        for algo, graph in (("bfs", g), ("sssp", gw)):
            fn = getattr(zc, algo)
            best = 1e9
            for _ in range(5):
                r = fn(graph, 0, s, collect_traffic=False, placement=placement)
                best = min(best, r.kernel_ms)
            te = r.total_traversed_edges
            eb = 8 if algo == "sssp" else 4
            print(f"{placement:8s} {algo:4s} {s.value:15s} iters={r.iterations:3d} "
                  f"kernel={best:8.3f} ms total={r.total_ms:8.3f} ms GTEPS={te/best/1e6:7.3f} "
                  f"linkGB/s={te*eb/best/1e6:7.2f} launches={r.launches}", flush=True)
        zc.release(graph)
