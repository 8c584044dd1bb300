"""A/B timing helper: median device time of every feasible format on a few
workloads (so_time_spmv: back-to-back multiplies, CUDA events) -- run twice
with and without a diagnostic knob (e.g. SOB_NO_CSR_COOP=1) to compare."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("AB_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6539.5
W = {"rmat": lambda: synth.rmat(22, 16, seed=42), "hyb": lambda: synth.hyb_skewed(4_000_000, 16, 160, 100, seed=6),
     "banded": lambda: synth.banded(4_000_000, 13, seed=2), "lap": lambda: synth.laplacian_2d(1000, seed=1),
     "unif": lambda: synth.uniform_random(4_000_000, 16, seed=4)}


def relabel(csr):
    """Columns renumbered by descending frequency (hot columns packed at the
    front of x), rows re-sorted: the same SpMV up to a permutation of x --
    a timing stand-in for hot-column packing."""
    freq = np.bincount(csr.col, minlength=csr.ncols)
    order = np.argsort(-freq, kind="stable")
    rank = np.empty(csr.ncols, dtype=np.int64)
    rank[order] = np.arange(csr.ncols)
    rows = np.repeat(np.arange(csr.nrows), np.diff(csr.row_ptr))
    nc = rank[csr.col]
    o = np.lexsort((nc, rows))
    return synth.HostCSR(csr.nrows, csr.ncols, csr.row_ptr, nc[o].astype(csr.col.dtype), csr.val[o])


W["rmat_rl"] = lambda: relabel(synth.rmat(22, 16, seed=42))
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for name in (sys.argv[2] if len(sys.argv) > 2 else "rmat,hyb,banded").split(","):
    csr = W[name]()
    base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    x = np.ones(csr.ncols)
    row = {}
    for f in range(6):
        try:
            m = base.convert(f)
        except P.PaddingOverflow:
            continue
        per, _ = m.time_spmv(x, 30)
        t = float(np.median(per))
        row[P.FORMAT_NAMES[f]] = f"{t * 1e6:.1f}us {m.spmv_bytes / t / 1e9 / PEAK:.3f}"
        del m
    print(tag, name, row, flush=True)
