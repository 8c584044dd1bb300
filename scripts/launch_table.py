#!/usr/bin/env python3
"""Per-launch table (sob kernels only) of an ncu --metrics launch-list CSV."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
s = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[s]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
per = defaultdict(dict)
for r in rows[s + 1:]:
    if len(r) < len(h):
        continue
    per[(int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0][-45:])][r[ix["Metric Name"]]] = float(
        r[ix["Metric Value"]].replace(",", ""))
for (i, k), m in sorted(per.items()):
    if "sob" in k or "unnamed" in k:
        b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        print(i, k, round(m["gpu__time_duration.sum"] / 1e3, 1), "us", round(b / 1e6, 1), "MB")
