"""A/B the expansion schedules / knobs on one K27 graph (zc_set_tuning specs)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--algo", default="bfs")
ap.add_argument("--configs", default="loop=host;;sched=chunk;unroll=8")
ap.add_argument("--strategy", default="merged-aligned")
ap.add_argument("--strategies", default="")
ap.add_argument("--pairs", action="store_true")
a = ap.parse_args()
t = time.time()
if a.algo == "sssp":
    dg = zc.generate_uniform_device(1 << a.scale, 16, 16, seed=27, weights=(8, 72))
else:
    dg = zc.generate_rmat(a.scale, 16, seed=27, symmetrize=a.algo == "cc")
print(f"gen {time.time()-t:.1f}s V={dg.num_vertices} E={dg.num_edges}", flush=True)
if a.pairs:
    dg.build_sssp_pairs()
if "compressed" in a.strategies:
    t = time.time()
    nb = dg.build_compressed()
    print(f"compressed {nb/1e9:.2f} GB = {nb/dg.num_edges:.2f} B/edge in {time.time()-t:.1f}s", flush=True)
src = int(zc.pick_sources(dg.as_csr(), 64, seed=7)[0])
eb = 8 if a.algo == "sssp" else 4
ref = None
runs = [(c, a.strategy) for c in a.configs.split(";")]
if a.strategies:
    runs = [("", s) for s in a.strategies.split(",")]
for cfg, strategy in runs:
    a.strategy = strategy
    dg.set_tuning(cfg)
    best = None
    for rep in range(3):
        r = zc.cc(dg, a.strategy, collect_traffic=False) if a.algo == "cc" else \
            getattr(zc, a.algo)(dg, src, a.strategy, collect_traffic=False)
        if best is None or r.kernel_ms < best.kernel_ms:
            best = r
    if ref is None:
        ref = best.values.copy()
    same = bool((best.values == ref).all())
    prof = dg.expand_profile(best.iterations)
    top = sorted(range(best.iterations), key=lambda k: -prof[k])[:3]
    lv = " ".join(f"L{k}:{best.traversed_edges[k]*eb/prof[k]/1e6:.1f}GB/s/{prof[k]:.1f}ms" for k in top)
    print(f"[{strategy} {cfg or 'default'}] iters={best.iterations} kernel={best.kernel_ms:.2f}ms "
          f"GTEPS={best.total_traversed_edges/best.kernel_ms/1e6:.3f} "
          f"link={best.total_traversed_edges*eb/best.expand_ms/1e6:.2f}GB/s same={same} | {lv}",
          flush=True)
