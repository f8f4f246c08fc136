"""Sum an ncu --csv launch list (gpu__time_duration, dram__bytes_read/write) into one JSON record.

  python tools/ncu_sum.py --key cfg1 --csv gpurun_out/smooth_cfg1.csv --out profiles/smooth_traffic.json
Used for bench.py's roofline.traffic: DRAM bytes of all kernels of one fine-level smooth
(tools/profile_kernel.py --which 5 --level 0, one launch bracketed by the profiler range).
"""
import argparse
import csv
import json
import os

ap = argparse.ArgumentParser()
ap.add_argument("--key", required=True)
ap.add_argument("--csv", required=True)
ap.add_argument("--out", required=True)
ap.add_argument("--divide", type=int, default=1,
                help="component launches in the profiled range (smg_time_kernel runs 1 warm-up + reps)")
a = ap.parse_args()
rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[1:]:
    per.setdefault(int(r[ii]), {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
kern = {}
tot_b = tot_us = 0.0
for m in per.values():
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    us = m.get("gpu__time_duration.sum", 0.0) / 1e3
    tot_b += b
    tot_us += us
    name = m["kernel"].split("(")[0].replace("void ", "")
    k = kern.setdefault(name, {"launches": 0, "dram_bytes": 0.0, "ncu_us": 0.0})
    k["launches"] += 1
    k["dram_bytes"] += b
    k["ncu_us"] += us
out = json.load(open(a.out)) if os.path.exists(a.out) else {}
out[a.key] = {"dram_bytes": tot_b / a.divide, "ncu_us_cold_serialised": tot_us / a.divide,
              "kernel_launches": len(per) / a.divide, "per_kernel_in_range": kern, "component_launches_in_range": a.divide,
              "source": os.path.basename(a.csv)}
json.dump(out, open(a.out, "w"), indent=1)
print(a.key, "launches", len(per) / a.divide, "dram GB", round(tot_b / a.divide / 1e9, 3),
      "ncu us", round(tot_us / a.divide, 1))
