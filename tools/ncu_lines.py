"""Per-source-line warp-stall samples of an ncu report's source page.

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_lines.py src.csv [--top 40] [--regions 1955:vel,2010:pf,...]
"""
import argparse
import collections
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--regions", default="")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = next(r for r in rows if r and r[0] == "Line No")
si, ii = hdr.index("# Samples"), hdr.index("Instructions Executed")
data = []
for r in rows:
    if len(r) <= si or not r[0].isdigit():
        continue
    try:  # source text with embedded quotes shifts the columns: index from the end
        data.append((int(r[0]), int(r[si - len(hdr)] or 0), int(r[ii - len(hdr)] or 0), r[1]))
    except ValueError:
        continue
tot = sum(d[1] for d in data) or 1
toti = sum(d[2] for d in data) or 1
print(f"total samples {tot}, warp instructions {toti}")
if a.regions:
    cuts = [(int(c.split(":")[0]), c.split(":")[1]) for c in a.regions.split(",")]
    agg, aggi = collections.Counter(), collections.Counter()
    for ln, s, n, _ in data:
        name = "<first"
        for lo, nm in cuts:
            if ln >= lo:
                name = nm
        agg[name] += s
        aggi[name] += n
    for k, v in agg.most_common():
        print(f"{k:24s} {v:8d} {100 * v / tot:5.1f}% samples   {100 * aggi[k] / toti:5.1f}% instructions")
print("--- top lines")
for ln, s, n, src in sorted(data, key=lambda t: -t[1])[: a.top]:
    print(f"{ln:5d} {s:7d} {100 * s / tot:5.1f}% {n:9d}  {src.strip()[:100]}")
