"""near-far SSSP: device time / work over the bucket width delta (U27 and a
weighted K27), merged-aligned and compressed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
for name, dg in (("U%d" % scale, lambda: zc.generate_uniform_device(1 << scale, 16, 16, seed=27,
                                                                     weights=(8, 72))),
                 ("K%d-w" % scale, lambda: zc.generate_rmat(scale, 16, seed=27, weights=(8, 72)))):
    g = dg()
    src = int(zc.pick_sources(g.as_csr(), 1, seed=7)[0])
    for strat in ("merged-aligned", "compressed"):
        for delta in (8, 16, 32, 64, 128, 256):
            best = None
            for _ in range(2):
                r = zc.sssp(g, src, strat, collect_traffic=False, schedule="near-far", delta=delta)
                if best is None or r.kernel_ms < best.kernel_ms:
                    best = r
            print(f"{name} {strat:15s} delta={delta:4d} iters={best.iterations:4d} "
                  f"work={best.total_traversed_edges / g.num_edges:.3f}E ms={best.kernel_ms:8.1f}",
                  flush=True)
    g.close()
