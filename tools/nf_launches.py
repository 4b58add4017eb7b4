"""One near-far SSSP on U27 inside an NVTX range "nf" (after a warm-up run),
for an ncu launch list of the iterations:
  ncu --nvtx --nvtx-include "nf/" --metrics gpu__time_duration.sum --csv \
      python tools/nf_launches.py --strategy compressed"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2006_06890_b200 as zc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--strategy", default="compressed")
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--delta", type=int, default=16)
args = ap.parse_args()
u = zc.generate_uniform_device(1 << args.scale, 16, 16, seed=1, weights=(8, 72))
src = int(zc.pick_sources(u.as_csr(), 1, seed=7)[0])
r = zc.sssp(u, src, args.strategy, schedule="near-far", delta=args.delta)
torch.cuda.nvtx.range_push("nf")
r = zc.sssp(u, src, args.strategy, schedule="near-far", delta=args.delta)
torch.cuda.nvtx.range_pop()
print(f"{args.strategy}: iterations={r.iterations} kernel_ms={r.kernel_ms:.2f} "
      f"expand_ms={r.expand_ms:.2f} frontiers={r.frontier_sizes} trav={r.traversed_edges}")
