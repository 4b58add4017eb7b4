"""Gather roofline of the in-HBM control run (zc_gather_probe): random 4-byte
loads into an L2-resident bitmap (16 MB = K27's visited bitmap) and into
larger arrays, with and without the claims' atomics."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200._native as N
for nbytes in (16 << 20, 64 << 20, 512 << 20):
    for mode in (0, 1):
        out = C.c_double()
        N.check(N.probe_lib().zc_gather_probe(0, nbytes, mode, C.byref(out)))
        print(f"{nbytes >> 20:5d} MB mode={mode} ({'loads' if mode == 0 else 'loads + 1/16 atomicOr'}): "
              f"{out.value:.1f} G random 4-byte loads/s", flush=True)
