"""Print the key metrics of ncu raw-page CSV exports (one kernel each)."""
import csv, sys
KEYS = ["gpu__time_duration.sum", "pcie__read_bytes.sum.per_second", "pcie__read_bytes.sum",
        "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum",
        "syslts__t_requests_srcunit_tex_aperture_sysmem_op_read.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, zip(vals, units)))
    print(f)
    for k in KEYS:
        if k in d:
            print(f"  {k:75s} {d[k][0]:>20s} {d[k][1]}")
    extra = [h for h in hdr if "syslts__t_requests" in h and "pct" not in h and "per_second" not in h]
    for k in extra[:6]:
        print(f"  {k:75s} {d[k][0]:>20s} {d[k][1]}")
