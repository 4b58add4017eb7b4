"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv): count, summed duration, share of the traversal kernels."""
import collections, csv, re, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    m = re.search(r"(k_\w+|cub::\w+|DeviceScan\w*|\w+Kernel\w*)", r[ki])
    name = m.group(1) if m else r[ki][:40]
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[ui], 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
trav = {k: v for k, v in tot.items() if k.startswith(("k_expand", "k_window", "k_tile", "k_level", "k_cand", "k_fbits", "k_narrow",
                                                     "k_init", "k_widen", "cub::DeviceScan",
                                                     "DeviceScan", "k_scan"))}
s = sum(trav.values())
print(f"{'kernel':36s} {'launches':>8s} {'total ms':>10s} {'share of traversal':>18s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    share = f"{v / s:.3f}" if k in trav else "-"
    print(f"{k:36s} {cnt[k]:8d} {v:10.2f} {share:>18s}")
