"""e2e breakdown of the bench's pipelined call: bfs_many over 10 K27 sources,
wall time vs summed device time, for several widen thread settings (env
ZC_WIDEN_SPARE is read once per process, so each setting runs in a child)."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2006_06890_b200 as zc
    dg = zc.generate_rmat(27, 16, seed=27)
    srcs = [int(s) for s in zc.pick_sources(dg.as_csr(), 64, seed=7)[3:13]]
    zc.bfs_many(dg, srcs, "direction-optimizing")
    for rep in range(2):
        t = time.perf_counter()
        rs = zc.bfs_many(dg, srcs, "direction-optimizing")
        wall = (time.perf_counter() - t) * 1e3
        k = sum(r.kernel_ms for r in rs)
        e = sum(r.total_traversed_edges for r in rs)
        print(f"spare={os.environ.get('ZC_WIDEN_SPARE','2')} wall={wall:.1f}ms kernel={k:.1f}ms "
              f"e2e={e/wall/1e6:.2f} GTEPS value={e/k/1e6:.2f}", flush=True)
        rs = None
    sys.exit(0)
for spare in sys.argv[1:] or ["2"]:
    env = dict(os.environ, ZC_WIDEN_SPARE=spare)
    subprocess.run([sys.executable, __file__, "child"], env=env)
