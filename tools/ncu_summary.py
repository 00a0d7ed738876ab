"""Summarize an ncu report (--set full) or a launch-list CSV into a small JSON + markdown table for
profiles/.  Usage:
    python tools/ncu_summary.py report.ncu-rep out_prefix [--algo-bytes-json file]
    python tools/ncu_summary.py --launches launches.csv out_prefix
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def _csv(cmd):
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows


def summarize_report(rep, prefix):
    rows = _csv(["ncu", "-i", rep, "--page", "raw", "--csv"])
    h, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(h)}

    def val(r, name, scale_to=None):
        i = col.get(name)
        if i is None or not r[i]:
            return None
        v = float(r[i].replace(",", ""))
        u = units[i]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1,
                "nsecond": 1e-9}.get(u, 1.0)
        return v * mult

    out = []
    for r in rows[2:]:
        stalls = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[i] or 0)
                  for n, i in col.items() if n.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not n.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda x: -x[1])[:4]
        t = val(r, "gpu__time_duration.sum")
        rd = val(r, "dram__bytes_read.sum") or 0.0
        wr = val(r, "dram__bytes_write.sum") or 0.0
        out.append({
            "kernel": r[col["Kernel Name"]],
            "duration_s": t,
            "dram_read_bytes": rd,
            "dram_write_bytes": wr,
            "dram_GBps": (rd + wr) / t / 1e9 if t else None,
            "dram_pct_peak": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "achieved_occupancy_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": val(r, "launch__registers_per_thread"),
            "grid": val(r, "launch__grid_size"),
            "block": val(r, "launch__block_size"),
            "top_stalls": [(k, round(100 * v / tot, 1)) for k, v in top],
        })
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"ncu --set full summary of `{rep}` (cold-cache, serialized replays)\n\n")
        f.write("| kernel | ms | DRAM read GB | DRAM write GB | GB/s | DRAM % peak | occ % | regs | top stalls % |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for o in out:
            f.write(f"| {o['kernel'][:60]} | {o['duration_s'] * 1e3:.3f} | {o['dram_read_bytes'] / 1e9:.3f} | "
                    f"{o['dram_write_bytes'] / 1e9:.3f} | {o['dram_GBps'] or 0:.0f} | {o['dram_pct_peak'] or 0:.1f} | "
                    f"{o['achieved_occupancy_pct'] or 0:.1f} | {int(o['registers'] or 0)} | "
                    f"{', '.join(f'{k} {v}' for k, v in o['top_stalls'])} |\n")
    return out


def summarize_launches(path, prefix):
    txt = open(path).read()
    lines = [ln for ln in txt.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(r[iu], 1.0)
        name = r[ik].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
        total += v
    out = {k: {"launches": n, "total_s": t, "share": t / total} for k, (n, t) in
           sorted(agg.items(), key=lambda x: -x[1][1])}
    json.dump({"total_s": total, "kernels": out}, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"ncu launch list `{path}` (gpu__time_duration.sum, cold-cache serialized): "
                f"{sum(v['launches'] for v in out.values())} launches, {total * 1e3:.2f} ms total\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, v in out.items():
            f.write(f"| {k} | {v['launches']} | {v['total_s'] * 1e3:.3f} | {100 * v['share']:.1f}% |\n")
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        r = summarize_launches(sys.argv[2], sys.argv[3])
    else:
        r = summarize_report(sys.argv[1], sys.argv[2])
    print(json.dumps(r, indent=1)[:3000])
