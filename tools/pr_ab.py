"""PageRank on K27-sym, merged-aligned, 5 iterations: default load flavour vs ld=1 (plain windows), interleaved."""
import sys, warnings
sys.path.insert(0, "/root/repo")
import paper_2006_06890_b200 as zc
warnings.simplefilter("ignore")
k = zc.generate_rmat(27, 16, seed=27, symmetrize=True)
for rnd in range(3):
    for spec in ("", "ld=1"):
        k.set_tuning(spec)
        zc.pagerank(k, "merged-aligned", max_iters=1, tol=1e-30, collect_traffic=False)
        r = zc.pagerank(k, "merged-aligned", max_iters=5, tol=1e-30, collect_traffic=False)
        print(rnd, spec or "default", round(r.total_traversed_edges / (r.kernel_ms * 1e-3) / 1e9, 3), flush=True)
