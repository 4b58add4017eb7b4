"""e2e of bfs_many (int64 results downloaded and widened on host threads while
the next traversal runs) over the widen thread count, per strategy (K27)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
dg = zc.generate_rmat(27, 16, seed=27)
srcs = [int(s) for s in zc.pick_sources(dg.as_csr(), 64, seed=7)[:24]]
for strat in ("direction-optimizing", "merged-aligned"):
    for rnd in range(2):
        for w in ("widen=2", "", "widen=8", "widen=12"):
            dg.set_tuning(w)
            zc.bfs_many(dg, srcs[:8], strat)
            t = time.perf_counter(); trav = dev = 0
            for b in range(0, 24, 8):
                for r in zc.bfs_many(dg, srcs[b:b + 8], strat):
                    trav += r.total_traversed_edges
                    dev += r.kernel_ms
            wall = time.perf_counter() - t
            if rnd:
                print(f"{strat:22s} {w or 'widen=4 (default)':18s} e2e {trav / wall / 1e9:6.2f} GTEPS, "
                      f"device {trav / dev / 1e6:6.2f}", flush=True)
