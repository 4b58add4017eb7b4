"""Sum ncu --metrics gpu__time_duration.sum CSV launch lists per kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi, ui, mi = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
agg = defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    if len(r) < len(hdr) or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    ms = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[ui], 1e-6) * v
    name = r[ki].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += ms
tot = sum(v[1] for v in agg.values())
for name, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{ms:10.2f} ms {100 * ms / tot:5.1f}% {n:6d}  {name}")
print(f"{tot:10.2f} ms total")
