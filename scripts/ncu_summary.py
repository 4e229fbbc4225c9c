"""Fold an `ncu --page raw --csv` capture into profiles/ncu_summary.json.

    python scripts/ncu_summary.py CONFIG RAW_CSV SOURCE_TEXT

Records, per launch: duration, DRAM read/write bytes, L2 hit rate, L2->SM
bytes, the busiest pipes and the binding resource (the largest of DRAM
throughput, L2 throughput and the busiest SM pipe, as ncu reports them).
"""
import csv
import json
import os
import sys

cfg, path, source = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
names, units = rows[hdr], rows[hdr + 1]
data = [r for r in rows[hdr + 2:] if len(r) == len(names)][-1]


def get(name, scale=1.0):
    i = names.index(name)
    v = data[i].replace(",", "")
    u = units[i]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "ms": 1e3, "us": 1, "ns": 1e-3, "msecond": 1e3, "usecond": 1}.get(u, 1)
    return float(v) * mult * scale


pipes = {n.split("sm__pipe_")[1].split("_cycles")[0]: float(data[i])
         for i, n in enumerate(names)
         if n.startswith("sm__pipe_") and n.endswith("cycles_active.avg.pct_of_peak_sustained_active")
         and data[i] not in ("", "n/a")}
top = sorted(pipes.items(), key=lambda kv: -kv[1])[:4]
dram_pct = get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
l2_pct = get("lts__throughput.avg.pct_of_peak_sustained_elapsed")
cands = {"hbm": dram_pct, "l2": l2_pct, f"{top[0][0]}-pipe": top[0][1]}
bound = max(cands, key=cands.get)
rec = {
    "kernel": data[names.index("Kernel Name")],
    "ncu_duration_us": get("gpu__time_duration.sum"),
    "dram_read_bytes": get("dram__bytes_read.sum"),
    "dram_write_bytes": get("dram__bytes_write.sum"),
    "l2_hit_pct": get("lts__t_sector_hit_rate.pct"),
    "l2_to_sm_bytes": get("l1tex__m_xbar2l1tex_read_bytes.sum"),
    "dram_throughput_pct": dram_pct,
    "l2_throughput_pct": l2_pct,
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers": get("launch__registers_per_thread"),
    "top_pipes_pct": dict(top),
    "bound": bound,
    "bound_pct": cands[bound],
    "source": source,
}
rec["dram_bytes_per_launch"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   "ncu_summary.json")
allrec = json.load(open(out)) if os.path.exists(out) else {}
allrec[cfg] = rec
json.dump(allrec, open(out, "w"), indent=1)
print(cfg, json.dumps(rec, indent=1))
