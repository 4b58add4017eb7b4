"""Line-compressed lists at scale: build time and size, then BFS (K27) and
CC (K27 symmetric) per level, compressed vs packed, results compared."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
algos = sys.argv[2].split(",") if len(sys.argv) > 2 else ["bfs", "cc"]
for algo in algos:
    t = time.time()
    if algo == "sssp":  # BASELINE configs[2]: uniform degree 16, u32 weights [8, 72]
        dg = zc.generate_uniform_device(1 << scale, 16, 16, seed=27, weights=(8, 72))
    else:
        dg = zc.generate_rmat(scale, 16, seed=27, symmetrize=algo == "cc")
    print(f"[{algo}] gen {time.time()-t:.1f}s V={dg.num_vertices} E={dg.num_edges}", flush=True)
    t = time.time()
    nb = dg.build_compressed()
    print(f"compressed stream {nb/2**30:.2f} GiB = {nb/dg.num_edges:.3f} B/edge (all edges) "
          f"in {time.time()-t:.1f}s", flush=True)
    src = int(zc.pick_sources(dg.as_csr(), 64, seed=7)[0])
    res = {}
    if algo == "sssp":
        dg.build_sssp_pairs()
    for s in ("packed", "compressed"):
        for rep in range(2):
            r = zc.cc(dg, s, collect_traffic=False) if algo == "cc" else \
                getattr(zc, algo)(dg, src, s, collect_traffic=False)
        res[s] = r
        prof = dg.expand_profile(r.iterations)
        print(f"== {algo} {s} iters={r.iterations} kernel={r.kernel_ms:.2f}ms "
              f"GTEPS={r.total_traversed_edges/r.kernel_ms/1e6:.3f} "
              f"u32-equiv-link={r.total_traversed_edges*(8 if algo == 'sssp' else 4)/r.expand_ms/1e6:.2f}GB/s",
              flush=True)
        print("   levels ms: " + " ".join(f"{p:.2f}" for p in prof[:r.iterations]), flush=True)
    a, b = res["packed"], res["compressed"]
    print("identical:", bool(np.array_equal(a.values, b.values)) and a.iterations == b.iterations
          and a.traversed_edges == b.traversed_edges, flush=True)
    dg.close()
