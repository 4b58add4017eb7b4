"""ZC_DEBUG_DO per-level trace of direction-optimizing BFS for chosen K27 sources."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
dg = zc.generate_rmat(27, 16, seed=27)
os.environ["ZC_DEBUG_DO"] = "1"
for a in sys.argv[2].split(","):
    os.environ["ZC_TUNE"] = f"do_alpha={a}"
    for s in [int(x) for x in sys.argv[1].split(",")]:
        zc.bfs(dg, s, "direction-optimizing", collect_traffic=False)
        print(f"--- src {s} alpha {a}", file=sys.stderr, flush=True)
        r = zc.bfs(dg, s, "direction-optimizing", collect_traffic=False)
        print(f"src {s} alpha {a} {r.kernel_ms:.1f} ms", file=sys.stderr, flush=True)
