"""Direction-optimizing BFS on K27: in-list build, per-level directions and
times beside the compressed top-down run, several switch factors; results
compared with the top-down run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
alphas = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2.0]
sym = len(sys.argv) > 3 and sys.argv[3] == "sym"
dg = zc.generate_rmat(scale, 16, seed=27, symmetrize=sym)
t = time.time()
nb = dg.build_compressed()
t1 = time.time()
nin = dg.build_in_lists()
print(f"V={dg.num_vertices} E={dg.num_edges} out-stream {nb/2**30:.2f} GiB ({t1-t:.1f}s) "
      f"in-stream {nin/2**30:.2f} GiB ({time.time()-t1:.1f}s)", flush=True)
srcs = [int(s) for s in zc.pick_sources(dg.as_csr(), 64, seed=7)[:6]]
for s in srcs[:1]:
    zc.bfs(dg, s, "compressed", collect_traffic=False)
    ref = zc.bfs(dg, s, "compressed", collect_traffic=False)
    prof = dg.expand_profile(ref.iterations)
    print(f"compressed src={s} {ref.kernel_ms:.2f} ms GTEPS={ref.total_traversed_edges/ref.kernel_ms/1e6:.2f} "
          f"levels: " + " ".join(f"{p:.2f}" for p in prof), flush=True)
for a in alphas:
    dg.set_tuning(f"do_alpha={a}")
    tot_e = tot_ms = 0
    for s in srcs:
        zc.bfs(dg, s, "direction-optimizing", collect_traffic=False)
        r = zc.bfs(dg, s, "direction-optimizing", collect_traffic=False)
        tot_e += r.total_traversed_edges
        tot_ms += r.kernel_ms
        same = None
        if s == srcs[0]:
            same = (np.array_equal(r.values, ref.values) and r.iterations == ref.iterations
                    and r.traversed_edges == ref.traversed_edges)
        if True:
            prof = dg.expand_profile(r.iterations)
            d = dg.directions(r.iterations)
            print(f"DO alpha={a} src={s} {r.kernel_ms:.2f} ms "
                  f"GTEPS={r.total_traversed_edges/r.kernel_ms/1e6:.2f} same={same} "
                  f"trav={r.total_traversed_edges} levels: "
                  + " ".join(f"{p:.2f}{'^' if x else ''}" for p, x in zip(prof, d)), flush=True)
    print(f"DO alpha={a}: {len(srcs)} sources mean GTEPS {tot_e/tot_ms/1e6:.2f}", flush=True)
