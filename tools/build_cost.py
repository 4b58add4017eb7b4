"""Cost of the compressed out-list and in-list builds at K27 (VERDICT r01
item 7): wall time of each build call, plus the pinned-allocation cost of
the same byte counts on its own.  Run plain, then under ncu --metrics
gpu__time_duration.sum for the kernel share."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
import paper_2006_06890_b200._native as N
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
t = time.time()
dg = zc.generate_rmat(scale, 16, seed=27)
print(f"gen {time.time() - t:.2f}s", flush=True)
t = time.time()
nb = dg.build_compressed()
print(f"build_compressed {time.time() - t:.2f}s bytes={nb}", flush=True)
t = time.time()
ni = dg.build_in_lists()
print(f"build_in_lists {time.time() - t:.2f}s bytes={ni}", flush=True)
print("phases (ms):", " ".join(f"{k}={v:.0f}" for k, v in dg.build_log()), flush=True)
for nbytes in (nb, ni):
    t = time.time()
    p = N.lib().zc_host_alloc(nbytes)
    ta = time.time() - t
    t = time.time()
    N.lib().zc_host_free(p)
    print(f"zc_host_alloc({nbytes}) {ta:.2f}s free {time.time() - t:.2f}s", flush=True)
dg.close()
# a fresh graph's direction-optimizing build in one call: the out-list sort's
# first radix transpose is kept as the in-lists (no second transpose)
for tune in ("", "sort=segmented"):
    dg = zc.generate_rmat(scale, 16, seed=27)
    dg.set_tuning(tune)
    t = time.time()
    ni = dg.build_in_lists()
    print(f"[{tune or 'sort=radix'}] fresh build_in_lists (out + in) {time.time() - t:.2f}s "
          f"bytes={ni}", flush=True)
    print("phases (ms):", " ".join(f"{k}={v:.0f}" for k, v in dg.build_log()), flush=True)
    dg.close()
