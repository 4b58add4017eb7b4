"""zerocopy-managed placement: small parity vs the oracle, then K27 BFS per
level beside pinned zero-copy, with the HBM use before / after (the lists
must stay in host memory)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_2006_06890_b200 as zc

g = zc.with_uniform_weights(zc.generate_uniform(4096, 4, 24, seed=3))
src = int(zc.pick_sources(g, 1)[0])
for s in ("naive", "merged", "merged-aligned", "packed"):
    assert np.array_equal(zc.bfs(g, src, s, collect_traffic=False, placement="zerocopy-managed").values,
                          oracle.bfs(g, src).values)
    assert np.array_equal(zc.sssp(g, src, s, collect_traffic=False, placement="zerocopy-managed").values,
                          oracle.sssp(g, src).values)
print("small parity ok", flush=True)
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
for placement in ("zerocopy-managed", "zerocopy"):
    f0 = torch.cuda.mem_get_info(0)[0]
    t = time.time()
    dg = zc.generate_rmat(scale, 16, seed=27, placement=placement)
    f1 = torch.cuda.mem_get_info(0)[0]
    print(f"[{placement}] gen {time.time()-t:.1f}s hbm used by handle {(f0-f1)/2**30:.2f} GiB", flush=True)
    srcs = zc.pick_sources(dg.as_csr(), 64, seed=7)
    src = int(srcs[0])
    for s in ("packed", "merged-aligned", "merged"):
        for rep in range(2):
            r = zc.bfs(dg, src, s, collect_traffic=False)
        prof = dg.expand_profile(r.iterations)
        print(f"== {placement} bfs {s} kernel={r.kernel_ms:.2f}ms GTEPS={r.total_traversed_edges/r.kernel_ms/1e6:.3f} "
              f"link={r.total_traversed_edges*4/r.expand_ms/1e6:.2f}GB/s", flush=True)
        print("   levels ms: " + " ".join(f"{p:.2f}" for p in prof[:r.iterations]), flush=True)
    ts = []
    for sv in srcs[:8]:
        r = zc.bfs(dg, int(sv), "packed", collect_traffic=False)
        ts.append(r.total_traversed_edges / r.kernel_ms / 1e6)
    f2 = torch.cuda.mem_get_info(0)[0]
    print(f"[{placement}] packed 8-source mean GTEPS {np.mean(ts):.3f}; hbm delta after runs "
          f"{(f1-f2)/2**30:.2f} GiB", flush=True)
    if placement == "zerocopy-managed":
        ref = oracle.bfs(dg.as_csr(), src, threads=os.cpu_count())
        r = zc.bfs(dg, src, "packed", collect_traffic=False)
        print("K bit-exact vs oracle:", bool(np.array_equal(r.values, ref.values)), flush=True)
    dg.close()
