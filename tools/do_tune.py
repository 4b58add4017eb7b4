"""Direction-optimizing BFS mean GTEPS (16 K27 sources) under ZC_TUNE variants."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc

dg = zc.generate_rmat(27, 16, seed=27, placement=os.environ.get("PLACEMENT", "zerocopy"))
srcs = [int(s) for s in zc.pick_sources(dg.as_csr(), 64, seed=7)[:16]]
zc.bfs(dg, srcs[0], "direction-optimizing", collect_traffic=False)
for tune in sys.argv[1:]:
    dg.set_tuning(tune)
    e = ms = 0
    for s in srcs:
        r = zc.bfs(dg, s, "direction-optimizing", collect_traffic=False)
        e += r.total_traversed_edges
        ms += r.kernel_ms
    print(f"{tune!r}: mean GTEPS {e/ms/1e6:.2f}", flush=True)
