"""Top SASS instructions by warp-stall samples from `ncu -i rep --page source --csv --print-source sass`
output (one kernel).  Usage: python tools/ncu_sass_hot.py sass.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
isrc, iss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[iss] or 0), r[isrc].strip()))
    except (ValueError, IndexError):
        continue
tot = sum(x for x, _ in data) or 1.0
for i, (x, s) in enumerate(data):
    pass
order = sorted(range(len(data)), key=lambda i: -data[i][0])[:n]
for i in sorted(order):
    print(f"{i:5d} {100 * data[i][0] / tot:5.1f}%  {data[i][1][:100]}")
