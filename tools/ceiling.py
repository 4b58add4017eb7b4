"""Per-level ceiling model of the merged / merged-aligned BFS (VERDICT r01
item 4): the reference's request model (coalesce.py:165-207, evaluated on the
GPU for the same frontiers) times the measured per-size zero-copy request
rates (CTA-streamed reads of 32/64/96/128-byte chunks), next to the measured
per-level expansion time.

  ceiling_ms(level) = sum_c  n_c * c / rate_c      (c = 32, 64, 96, 128 B)

n_c = modelled requests of c bytes (edges; BFS reads no weights); rate_c =
GB/s of the probe at chunk size c.  ratio = ceiling / measured: 1.0 = the
kernel runs at the link's rate for its request mix; > 1 means the hardware
issued fewer requests than the model (L1 hits on lines shared by adjacent
lists).  Development / evidence tool (profiles/r02_ceiling_model.txt)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc
from paper_2006_06890_b200.device import read_probe

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--sources", type=int, default=3)
ap.add_argument("--strategies", default="merged-aligned,merged")
ap.add_argument("--algo", default="bfs", choices=["bfs", "sssp", "cc"])
a = ap.parse_args()
rates = {c: read_probe(1 << 30, c, 3, "pinned") for c in (32, 64, 96, 128)}
print("# probe: CTA-streamed zero-copy reads, GB/s per chunk size: "
      + " ".join(f"{c}B={g:.2f} ({g / c:.3f} G req/s)" for c, g in rates.items()), flush=True)
t = time.time()
if a.algo == "sssp":  # the bench's U27 (weights 8..72), separate arrays as the reference's model
    dg = zc.generate_uniform_device(1 << a.scale, 16, 16, seed=27, weights=(8, 72))
    dg.set_tuning("pairs=0")
    gname = "uniform"
else:
    dg = zc.generate_rmat(a.scale, 16, seed=27, symmetrize=a.algo == "cc")
    gname = "Kronecker" + (" symmetrized" if a.algo == "cc" else "")
print(f"# {a.algo} on {gname} {a.scale}: V={dg.num_vertices} E={dg.num_edges} "
      f"(gen {time.time() - t:.1f}s)", flush=True)
srcs = [int(s) for s in zc.pick_sources(dg.as_csr(), 64, seed=7)[:a.sources]]
if a.algo == "cc":
    srcs = srcs[:1]
run = {"bfs": lambda s, src, m: zc.bfs(dg, src, s, collect_traffic=m),
       "sssp": lambda s, src, m: zc.sssp(dg, src, s, collect_traffic=m),
       "cc": lambda s, src, m: zc.cc(dg, s, collect_traffic=m)}[a.algo]
eb = 8 if a.algo == "sssp" else 4
print(f"{'strategy':15s} {'src':>10s} {'lvl':>3s} {'edges':>11s} {'req32':>10s} {'req64':>10s} "
      f"{'req96':>10s} {'req128':>10s} {'payload/useful':>14s} {'meas_ms':>9s} {'ceil_ms':>9s} "
      f"{'ratio':>6s} {'GB/s(4B/edge)':>13s}")
tot = {}
for s in a.strategies.split(","):
    for src in srcs:
        best = None
        for _ in range(2):
            r = run(s, src, False)
            if best is None or r.kernel_ms < best.kernel_ms:
                best = r
                prof = dg.expand_profile(r.iterations)
        m = run(s, src, True)
        assert m.iterations == best.iterations
        sm = tot.setdefault(s, [0.0, 0.0, 0.0])
        for k in range(best.iterations):
            h = m.per_iteration_traffic[k].hist  # edges (+ weights for SSSP: same windows)
            ceil = sum(h[c] * c / (rates[c] * 1e9) for c in (32, 64, 96, 128)) * 1e3
            e = best.traversed_edges[k]
            pay = sum(h[c] * c for c in (32, 64, 96, 128))
            meas = float(prof[k])
            big = e > 1e7
            if big:
                sm[0] += meas
                sm[1] += ceil
            sm[2] += meas
            print(f"{s:15s} {src:10d} {k:3d} {e:11d} {h[32]:10d} {h[64]:10d} {h[96]:10d} "
                  f"{h[128]:10d} {pay / max(eb * e, 1):14.3f} {meas:9.3f} {ceil:9.3f} "
                  f"{ceil / max(meas, 1e-9):6.3f} {eb * e / max(meas, 1e-9) / 1e6:13.2f}"
                  + ("" if big else "  (< 1e7 edges)"), flush=True)
        print(f"{s:15s} {src:10d} all GTEPS={best.total_traversed_edges / best.kernel_ms / 1e6:.3f} "
              f"kernel_ms={best.kernel_ms:.2f} expand_ms={best.expand_ms:.2f}", flush=True)
for s, (meas, ceil, alls) in tot.items():
    print(f"# {s}: levels > 1e7 edges: measured {meas:.1f} ms vs ceiling {ceil:.1f} ms "
          f"(ratio {ceil / meas:.3f}); all levels measured {alls:.1f} ms")
