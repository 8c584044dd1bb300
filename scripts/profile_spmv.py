"""Launch-list driver for ncu: every format's SpMV on a workload, a few
times each, then one feature extraction + tune.  Not a benchmark (numbers
printed under ncu are never bench values).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/launches.csv \
        python scripts/profile_spmv.py --workload banded
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="banded")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--formats", default="0,1,2,3,4,5")
    a = ap.parse_args()
    csr = {"banded": lambda: synth.banded(4_000_000, 13, seed=2),
           "laplacian": lambda: synth.laplacian_2d(1000, seed=1),
           "rmat": lambda: synth.rmat(22, 16, seed=42),
           "hyb": lambda: synth.hyb_skewed(4_000_000, 16, 160, 100, seed=6)}[a.workload]()
    base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    x = np.ones(csr.ncols)
    for f in [int(v) for v in a.formats.split(",")]:
        try:
            m = base.convert(f)
        except P.PaddingOverflow:
            print(P.FORMAT_NAMES[f], "infeasible")
            continue
        per, _ = m.time_spmv(x, a.reps)
        print(P.FORMAT_NAMES[f], "bytes", m.spmv_bytes, "ms", per.min() * 1e3)
        fv = m.extract_features(0.2)
        print("  features", fv.to_row())


if __name__ == "__main__":
    main()
