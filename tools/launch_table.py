"""Per-kernel table of an ncu --csv launch list (metrics gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum): launches, summed time, share, DRAM bytes and GB/s per kernel name.

  python tools/launch_table.py gpurun_out/launches.csv [--top 25]
"""
import argparse
import csv
import collections

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[1:]:
    per.setdefault(int(r[ii]), {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for m in per.values():
    name = m["kernel"].split("(")[0].replace("void ", "").replace("smg::<unnamed>::", "")
    us = m.get("gpu__time_duration.sum", 0.0) / 1e3
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    agg[name][0] += 1
    agg[name][1] += us
    agg[name][2] += b
    tot += us
print(f"{len(per)} launches, {tot / 1e3:.3f} ms summed (cold caches, serialised)")
print(f"{'kernel':40s} {'n':>5s} {'ms':>8s} {'share':>6s} {'GB':>8s} {'GB/s':>7s}")
for name, (n, us, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: a.top]:
    print(f"{name[:40]:40s} {n:5d} {us / 1e3:8.3f} {100 * us / tot:5.1f}% {b / 1e9:8.3f} {b / (us * 1e-6) / 1e9 if us else 0:7.0f}")
