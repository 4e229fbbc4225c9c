"""Print selected metrics of an `ncu --page raw --csv` export (one kernel)."""
import csv
import re
import sys

path = sys.argv[1]
pats = sys.argv[2:] or [r"gpu__time_duration.sum$", r"dram__bytes_(read|write).sum$",
                         r"lts__t_sector_hit_rate.pct$", r"sm__inst_executed_pipe_.*\.sum$",
                         r"sm__pipe_.*cycles_active.avg.pct_of_peak_sustained_active$",
                         r"sm__throughput.avg.pct", r"l1tex__m_xbar2l1tex_read_bytes.sum$",
                         r"smsp__issue_active.avg.pct", r"launch__registers_per_thread$",
                         r"sm__warps_active.avg.pct", r"lts__t_bytes.sum$",
                         r"smsp__average_warp_latency_issue_stalled|smsp__pcsamp_warps_issue_stalled_.*[^t]$"]
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "ID" in r[:2] or "Kernel Name" in r)
names, units = rows[hdr], rows[hdr + 1]
for r in rows[hdr + 2:]:
    if len(r) != len(names):
        continue
    print("kernel:", r[names.index("Kernel Name")][:120])
    for i, (n, u) in enumerate(zip(names, units)):
        if any(re.search(p, n) for p in pats):
            v = r[i]
            if v in ("", "0", "0.00", "n/a"):
                continue
            print(f"  {n:80s} {u:12s} {v}")
