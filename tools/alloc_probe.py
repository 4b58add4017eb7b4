"""Zero-copy read rate by host allocation kind: does a larger GPU mapping
granularity (VMM host-NUMA allocation, hugetlbfs, managed-on-host) lift the
random-line rate that bounds the tiny-list BFS levels?"""
import ctypes as C
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200._native as N
import paper_2006_06890_b200.device as d

size = int(sys.argv[1]) if len(sys.argv) > 1 else 8 << 30
print(subprocess.run("grep -i huge /proc/meminfo; cat /sys/kernel/mm/transparent_hugepage/enabled",
                     shell=True, capture_output=True, text=True).stdout, flush=True)
g = C.c_uint64()
rc = N.probe_lib().zc_vmm_host_probe(0, 1 << 30, C.byref(g))
print("vmm host granularity", g.value, "rc", rc, N.lib().zc_last_error().decode() if rc else "",
      flush=True)
if os.geteuid() == 0:
    try:
        with open("/proc/sys/vm/nr_hugepages", "w") as fh:
            fh.write(str((size >> 21) + 64))
    except OSError as e:
        print("nr_hugepages write failed:", e)
    print(open("/proc/sys/vm/nr_hugepages").read().strip(), "hugepages reserved", flush=True)
for alloc in ("pinned", "vmm", "hugetlb", "managed_host", "thp"):
    for random in (False, True):
        row = []
        for chunk in (128, 512):
            try:
                row.append(f"{chunk}B:{d.read_probe(size, chunk, random, alloc):6.2f}")
            except Exception as e:  # noqa: BLE001
                row.append(f"{chunk}B: err {e}")
        print(f"{alloc:12s} {'random' if random else 'seq':6s} " + " ".join(row), flush=True)
for alloc in ("pinned", "vmm"):
    print(f"{alloc:12s} random-1GiB 128B:{d.read_probe(1 << 30, 128, True, alloc):6.2f}", flush=True)
if os.geteuid() == 0:
    with open("/proc/sys/vm/nr_hugepages", "w") as fh:
        fh.write("0")
