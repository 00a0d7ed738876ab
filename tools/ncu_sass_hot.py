"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.
Usage: python tools/ncu_sass_hot.py report.ncu-rep <kernel-substring> [N]
(runs `ncu -i report --page source --csv --print-source sass`, keeps the first kernel whose name
contains the substring, prints the N hottest instructions with their main stall reasons)."""
import csv
import io
import subprocess
import sys

rep, sub = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, errors="replace").stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = r
    elif cur is not None:
        cur[2].append(r)
blk = next(b for b in blocks if sub in b[0])
h, data = blk[1], blk[2]
isrc, iss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, name in enumerate(h) if name.startswith("stall_") and "Not Issued" not in name]
tot = sum(float(r[iss] or 0) for r in data) or 1.0
order = sorted(range(len(data)), key=lambda i: -float(data[i][iss] or 0))[:n]
print(blk[0], f"total samples {tot:.0f}")
for i in sorted(order):
    r = data[i]
    st = sorted(((float(r[c] or 0), h[c][6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{i:5d} {100 * float(r[iss] or 0) / tot:5.1f}%  {r[isrc].strip()[:60]:60s} " +
          " ".join(f"{nm}={v:.0f}" for v, nm in st if v > 0))
