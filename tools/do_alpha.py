"""Mean direction-optimizing GTEPS over the bench's first 16 sources for
several switch factors (zc_set_tuning do_alpha=X), K27."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc

dg = zc.generate_rmat(27, 16, seed=27)
srcs = [int(s) for s in zc.pick_sources(dg.as_csr(), 64, seed=7)[:16]]
zc.bfs(dg, srcs[0], "direction-optimizing", collect_traffic=False)
for a in [float(x) for x in sys.argv[1].split(",")]:
    dg.set_tuning(f"do_alpha={a}")
    e = ms = 0
    per = []
    for s in srcs:
        r = zc.bfs(dg, s, "direction-optimizing", collect_traffic=False)
        e += r.total_traversed_edges
        ms += r.kernel_ms
        per.append(r.kernel_ms)
    print(f"alpha={a}: mean GTEPS {e/ms/1e6:.2f}  per-source ms: " + " ".join(f"{x:.0f}" for x in per),
          flush=True)
