"""Afforest CC on K27-sym: sampling-pass width over the compressed lists
(zc_set_tuning uf_sample) and merged-aligned beside it; values are checked
against the first run.  python tools/uf_sample_ab.py [--scale 27]"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2006_06890_b200 as zc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
k = zc.generate_rmat(args.scale, 16, seed=1, symmetrize=True)
base = zc.cc(k, "merged-aligned", schedule="afforest")
E = k.num_edges
print(f"K{args.scale}-sym arcs={E}")
rows = [("merged-aligned", "")] + [("compressed", f"uf_sample={w}") for w in (1, 2, 4, 8, 16, 96)]
for strat, tune in rows:
    k.set_tuning(tune)
    best = None
    for _ in range(args.reps):
        r = zc.cc(k, strat, schedule="afforest")
        assert np.array_equal(r.values, base.values), (strat, tune)
        best = r if best is None or r.kernel_ms < best.kernel_ms else best
    ms = best.kernel_ms
    print(f"{strat:15s} {tune or 'default':14s} kernel_ms={ms:8.2f} passes={best.iterations} "
          f"pass_elems={list(best.traversed_edges)} expand_ms={best.expand_ms:.2f} "
          f"primary_gteps={E / ms / 1e6:.2f}")
k.set_tuning("")
