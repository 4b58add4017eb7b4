"""Per-level top-down vs direction-optimizing times for chosen K27 sources
(frontier size, frontier out-edges, unvisited in-edges estimate)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc

dg = zc.generate_rmat(27, 16, seed=27)
g = dg.as_csr()
indeg = np.bincount(g.edges, minlength=g.num_vertices)
E = g.num_edges
for s in [int(x) for x in sys.argv[1].split(",")]:
    r = zc.bfs(dg, s, "compressed", collect_traffic=False)
    r = zc.bfs(dg, s, "compressed", collect_traffic=False)
    td = dg.expand_profile(r.iterations)
    lv = r.values
    print(f"src {s}: compressed {r.kernel_ms:.1f} ms", flush=True)
    mu = E - indeg[s]
    for k in range(r.iterations):
        f = lv == k
        print(f"  it {k} front={int(f.sum()):10d} trav={r.traversed_edges[k]:11d} m_u={int(mu):11d} "
              f"ratio={r.traversed_edges[k]/max(mu,1):7.3f} td={td[k]:7.2f} ms", flush=True)
        mu -= int(indeg[lv == k + 1].sum())
    for a in (0.5, 1, 2, 4):
        dg.set_tuning(f"do_alpha={a}")
        r = zc.bfs(dg, s, "direction-optimizing", collect_traffic=False)
        p = dg.expand_profile(r.iterations)
        d = dg.directions(r.iterations)
        print(f"  DO a={a}: {r.kernel_ms:.1f} ms  " + " ".join(f"{x:.2f}{'^' if y else ''}" for x, y in zip(p, d)), flush=True)
