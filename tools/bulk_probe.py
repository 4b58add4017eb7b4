"""TMA bulk-copy streaming reads from pinned host memory vs SM loads vs memcpy."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
from paper_2006_06890_b200 import _native as N

size = 4 << 30
print("link probe", zc.link_probe(nbytes=1 << 30, iters=5), flush=True)
for ctas in (1, 2, 4, 8):
    row = []
    for chunk in (512, 1024, 2048, 4096, 8192, 16384, 32768):
        if chunk * 4 > 200 * 1024:
            continue
        out = C.c_double()
        rc = N.probe_lib().zc_bulk_probe(0, size, chunk, ctas, 3, C.byref(out))
        row.append(f"{chunk}B:{out.value:6.2f}" if rc == 0 else f"{chunk}B:err")
    print(f"ctas/SM={ctas}: " + " ".join(row), flush=True)
