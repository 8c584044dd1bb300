"""Diagnostic: SpMV time (CSR by default; formats and cases from argv) on near-banded matrices with a fraction of long
rows (synth.hyb_skewed variants), to separate the cost of row-length skew
from the cost of the stream itself.  Not a benchmark line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
CASES = [(16, 16, 100), (16, 32, 100), (16, 64, 100), (16, 160, 100), (16, 384, 100),
         (16, 160, 1000), (16, 160, 20), (27, 27, 100)]
fmts = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1").split(",")]
if len(sys.argv) > 2:  # e.g. "16:16:100,9:9:100" (short:long:every)
    CASES = [tuple(int(t) for t in c.split(":")) for c in sys.argv[2].split(",")]
for short, long, every in CASES:
    c = synth.hyb_skewed(4_000_000, short, long, every, seed=6)
    base = P.DeviceMatrix.csr(c.nrows, c.ncols, c.row_ptr, c.col, c.val)
    x = np.ones(c.ncols)
    for f in fmts:
        try:
            m = base.convert(f)
        except P.PaddingOverflow:
            continue
        per, _ = m.time_spmv(x, 30)
        t = float(np.median(per[5:]))
        print(f"short={short:3d} long={long:4d} every={every:5d} {P.FORMAT_NAMES[f]} z={c.nnz} "
              f"{t*1e6:8.1f} us {m.spmv_bytes/t/1e9:7.0f} GB/s frac {m.spmv_bytes/t/1e9/PEAK:.3f}", flush=True)
        del m
    del base, c
