#!/usr/bin/env python3
"""Summaries of ncu output for profiles/.

  launches <csv>  per-kernel table from a --metrics launch list (share of GPU
                  time, per-launch DRAM bytes)
  full <ncu-rep>  key metrics of a --set full capture (duration, DRAM
                  traffic, throughput %, occupancy, top stall reasons)
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    per = defaultdict(dict)
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        per[(int(r[ix["ID"]]), r[ix["Kernel Name"]])][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in per.items():
        short = name.split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
        short = short.split("::")[-1] if "::" in short else short
        a = agg[short]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total us | share | avg us/launch | DRAM MB/launch |", "|---|---|---|---|---|---|"]
    for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {c} | {t / 1e3:.1f} | {t / total * 100:.1f}% | {t / c / 1e3:.1f} | {b / c / 1e6:.1f} |")
    return "\n".join(out)


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = r[0], r[1], r[2]
    out = [f"kernel: {vals[hdr.index('Kernel Name')][:100]}", "", "| metric | value | unit |", "|---|---|---|"]
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            out.append(f"| {w} | {vals[i]} | {units[i]} |")
    stalls = [(hdr[i][33:], float(vals[i] or 0)) for i in range(len(hdr))
              if "smsp__pcsamp_warps_issue_stalled" in hdr[i] and not hdr[i].endswith("not_issued")]
    tot = sum(v for _, v in stalls) or 1.0
    out += ["", "top stall reasons (pc sampling):", ""]
    for n, v in sorted(stalls, key=lambda t: -t[1])[:6]:
        out.append(f"- {n}: {v / tot * 100:.1f}%")
    return "\n".join(out)


def traffic(path, kernel, out_json):
    """Record DRAM read+write bytes per launch of `kernel` (from a full capture)
    into profiles/traffic.json for bench.py's roofline.traffic."""
    import json
    import os
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = r[0], r[1], r[2]

    def val(name):
        v = float(vals[hdr.index(name)].replace(",", ""))
        u = units[hdr.index(name)].lower()
        return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)

    b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    d = json.load(open(out_json)) if os.path.exists(out_json) else {}
    d[kernel] = int(b)
    json.dump(d, open(out_json, "w"), indent=1)
    return f"{kernel}: {b / 1e6:.1f} MB per launch"


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        print(traffic(sys.argv[2], sys.argv[3], sys.argv[4]))
    else:
        print(launches(sys.argv[2]) if sys.argv[1] == "launches" else full(sys.argv[2]))
