"""Interleaved A/B of tuning specs over several sources (K27 BFS): mean GTEPS
per spec, each (spec, source) run `reps` times in alternation."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--strategy", default="merged-aligned")
ap.add_argument("--specs", default=";unroll=8")
ap.add_argument("--sources", type=int, default=6)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--algo", default="bfs")
ap.add_argument("--placement", default="zerocopy")
a = ap.parse_args()
if a.algo == "sssp":
    dg = zc.generate_uniform_device(1 << a.scale, 16, 16, seed=27, weights=(8, 72),
                                    placement=a.placement)
else:
    dg = zc.generate_rmat(a.scale, 16, seed=27, symmetrize=a.algo == "cc", placement=a.placement)
srcs = [int(s) for s in zc.pick_sources(dg.as_csr(), 64, seed=7)[:a.sources]]
if a.algo == "cc":
    srcs = srcs[:1]
specs = a.specs.split(";")
tot = {s: [0, 0.0] for s in specs}
# blocks per spec (a tuning change rebuilds the level-loop graph), alternated
for rnd in range(a.rounds):
    for spec in (specs if rnd % 2 == 0 else specs[::-1]):
        dg.set_tuning(spec)
        zc.bfs(dg, srcs[0], a.strategy, collect_traffic=False) if a.algo == "bfs" else None
        for src in srcs:
            r = (zc.cc(dg, a.strategy, collect_traffic=False) if a.algo == "cc" else
                 getattr(zc, a.algo)(dg, src, a.strategy, collect_traffic=False))
            if rnd > 0 or a.rounds == 1:  # round 0 warms
                tot[spec][0] += r.total_traversed_edges
                tot[spec][1] += r.kernel_ms
for spec, (e, ms) in tot.items():
    print(f"[{spec or 'default'}] GTEPS={e / ms / 1e6:.3f} over {len(srcs)} sources x {a.rounds - 1} rounds",
          flush=True)
