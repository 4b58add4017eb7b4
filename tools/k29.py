"""K29 on ONE B200: Kronecker scale 29 symmetrized (2^34 arcs, 64 GiB of u32
lists in pinned host memory, u64 offsets), BFS + CC over zero-copy, checked
bit-exact against the oracle port.  SURVEY.md §8d names K29 as the multi-GPU
config; this shows one GPU already holds and streams it.  Development tool."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=29)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--strategies", default="packed,merged-aligned")
ap.add_argument("--cc", action="store_true")
ap.add_argument("--no-oracle", action="store_true")
a = ap.parse_args()

t = time.time()
dg = zc.generate_rmat(a.scale, a.ef, seed=29, symmetrize=True)
print(f"gen {time.time()-t:.1f}s V={dg.num_vertices} E={dg.num_edges} "
      f"({dg.num_edges*4/2**30:.0f} GiB u32 lists pinned)", flush=True)
g = dg.as_csr()
src = int(zc.pick_sources(g, 64, seed=7)[0])
results = {}
for s in a.strategies.split(","):
    for rep in range(2):
        r = zc.bfs(dg, src, s, collect_traffic=False)
    results[s] = r
    print(f"bfs {s:15s} src={src} iters={r.iterations} kernel={r.kernel_ms:.1f}ms "
          f"GTEPS={r.total_traversed_edges/r.kernel_ms/1e6:.3f} "
          f"link={r.total_traversed_edges*4/r.expand_ms/1e6:.2f}GB/s", flush=True)
if not a.no_oracle:
    import oracle
    t = time.time()
    ref = oracle.bfs(g, src, threads=os.cpu_count())
    print(f"oracle bfs {time.time()-t:.1f}s", flush=True)
    for s, r in results.items():
        print(f"  {s}: same={np.array_equal(ref.values, r.values)} "
              f"trav_same={ref.traversed_edges == list(r.traversed_edges)}", flush=True)
if a.cc:
    r = zc.cc(dg, "packed", collect_traffic=False)
    print(f"cc packed iters={r.iterations} kernel={r.kernel_ms:.1f}ms "
          f"work-GTEPS={r.total_traversed_edges/r.kernel_ms/1e6:.3f} "
          f"link={r.total_traversed_edges*4/r.expand_ms/1e6:.2f}GB/s", flush=True)
    if not a.no_oracle:
        t = time.time()
        ref = oracle.cc(g, threads=os.cpu_count())
        print(f"oracle cc {time.time()-t:.1f}s same={np.array_equal(ref.values, r.values)}",
              flush=True)
