"""Per-level breakdown of one traversal (frontier size, traversed edges,
expansion-kernel time, achieved link GB/s).  Development tool."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--algo", default="bfs")
ap.add_argument("--strategies", default="merged-aligned,merged")
ap.add_argument("--placement", default="zerocopy")
ap.add_argument("--uniform", action="store_true")
ap.add_argument("--tuning", default="", help="zc_set_tuning spec, e.g. loop=host under ncu")
a = ap.parse_args()
t = time.time()
if a.algo == "sssp" and a.uniform:
    dg = zc.generate_uniform_device(1 << a.scale, 16, 16, seed=27, weights=(8, 72),
                                    placement=a.placement)
else:
    dg = zc.generate_rmat(a.scale, a.ef, seed=27, symmetrize=a.algo == "cc",
                          weights=(8, 72) if a.algo == "sssp" else None, placement=a.placement)
dg.set_tuning(a.tuning)
print(f"gen {time.time()-t:.1f}s V={dg.num_vertices} E={dg.num_edges}", flush=True)
src = int(zc.pick_sources(dg.as_csr(), 64, seed=7)[0])
eb = 8 if a.algo == "sssp" else 4
for s in a.strategies.split(","):
    for rep in range(2):
        if a.algo == "cc":
            r = zc.cc(dg, s, collect_traffic=False)
        else:
            r = getattr(zc, a.algo)(dg, src, s, collect_traffic=False)
    prof = dg.expand_profile(r.iterations)
    print(f"== {a.algo} {s} iters={r.iterations} kernel={r.kernel_ms:.2f}ms expand={r.expand_ms:.2f}ms "
          f"GTEPS={r.total_traversed_edges/r.kernel_ms/1e6:.3f} "
          f"link={r.total_traversed_edges*eb/r.expand_ms/1e6:.2f}GB/s", flush=True)
    for k in range(r.iterations):
        te = r.traversed_edges[k]
        print(f"  it {k:3d} front={r.frontier_sizes[k]:11d} edges={te:12d} expand={prof[k]:9.3f}ms "
              f"GB/s={te*eb/max(prof[k],1e-9)/1e6:7.2f}", flush=True)
