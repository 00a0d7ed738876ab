"""Markdown table of an ncu `--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv` log (one row per launch, per-family sums).  python tools/ncu_counters_md.py in.csv > out.md"""
import csv
import io
import json
import sys

PEAK = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])

txt = open(sys.argv[1]).read()
lines = [ln for ln in txt.splitlines() if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
launch = {}
for r in rows:
    key = (r["ID"], r["Kernel Name"])
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3,
             "ms": 1.0, "s": 1e3}[unit]
    launch.setdefault(key, {})[r["Metric Name"]] = v * scale


def fam(name):
    if name.startswith("void k_marg") or name.startswith("k_marg"):
        return "K2"
    if "k_huge_out" in name or "k_huge_y" in name:
        return "K4" if "k_huge_out<1>" in name or "<true>" in name else "K5"
    if "k_huge_fused" in name:
        return "K5"
    if "pipe" in name:
        pre = name.split("(")[0].rstrip(">").split(",")[-1].strip().rstrip(">")
        return "K4" if pre in ("1", "true") else "K5"
    return "other"


print("| # | kernel | ms | DRAM read GB | DRAM write GB | GB/s | of peak |")
print("|---|---|---|---|---|---|---|")
fams = {}
for i, ((lid, name), m) in enumerate(sorted(launch.items(), key=lambda x: int(x[0][0]))):
    ms = m.get("gpu__time_duration.sum", 0.0)
    rd = m.get("dram__bytes_read.sum", 0.0) / 1e9
    wr = m.get("dram__bytes_write.sum", 0.0) / 1e9
    gbs = (rd + wr) / (ms * 1e-3) if ms else 0.0
    short = name.split("(")[0].replace("void ", "")
    print(f"| {i} | {short} | {ms:.3f} | {rd:.3f} | {wr:.3f} | {gbs:.0f} | {gbs / PEAK:.2f} |")
    f = fams.setdefault(fam(name), [0.0, 0.0])
    f[0] += ms
    f[1] += rd + wr
print()
print("| family | ms (serialized sum) | DRAM GB | GB/s | of peak |")
print("|---|---|---|---|---|")
for k in sorted(fams):
    ms, gb = fams[k]
    print(f"| {k} | {ms:.2f} | {gb:.2f} | {gb / (ms * 1e-3):.0f} | {gb / (ms * 1e-3) / PEAK:.2f} |")
