"""Does earlier pinned-memory churn slow later zero-copy graphs?  SSSP-U27
packed: fresh vs after allocating / freeing many pinned buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc
from paper_2006_06890_b200 import _native as N

def run(tag):
    u = zc.generate_uniform_device(1 << 27, 16, 16, seed=27, weights=(8, 72))
    src = int(zc.pick_sources(u.as_csr(), 1, seed=7)[0])
    zc.sssp(u, src, "packed", collect_traffic=False)
    r = zc.sssp(u, src, "packed", collect_traffic=False)
    print(tag, f"{r.kernel_ms:.1f} ms", flush=True)
    u.close()

run("fresh")
run("second")
# churn: many 64 MiB pinned buffers, free every other one
lib = N.lib()
ptrs = [lib.zc_host_alloc(64 << 20) for _ in range(400)]
for p in ptrs[::2]:
    lib.zc_host_free(p)
run("after-churn")
for p in ptrs[1::2]:
    lib.zc_host_free(p)
run("after-free")
