"""Pinned-allocation cost by method (zc_pin_probe): the compressed streams'
builds pin ~6 GB each."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200._native as N
nb = int(float(sys.argv[1])) if len(sys.argv) > 1 else 6 << 30
for mode, name in ((0, "cudaHostAlloc"), (1, "mmap+THP+touch+register"), (2, "mmap+4K+touch+register"),
                   (3, "mmap+THP+register(no touch)")):
    for threads in ((1,) if mode in (0, 3) else (1, 8, 32)):
        a, r = C.c_double(), C.c_double()
        rc = N.probe_lib().zc_pin_probe(nb, mode, threads, C.byref(a), C.byref(r))
        print(f"{name:28s} threads={threads:2d} rc={rc} alloc+touch={a.value:.3f}s "
              f"register={r.value:.3f}s total={a.value + r.value:.3f}s "
              f"({nb / (a.value + r.value) / 1e9:.1f} GB/s)", flush=True)
