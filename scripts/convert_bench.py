"""Conversion cost CSR -> each format (switch_format's device path) and the
feature extraction, on configs 1-3: wall time per call (the conversions sync
on their size phases), median of 5 after a warm-up.  Diagnostic."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402


def bench(name, csr):
    base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    out = {}
    for f in range(6):
        ts = []
        try:
            for r in range(6):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                m = base.convert(f)
                torch.cuda.synchronize()
                if r:
                    ts.append(time.perf_counter() - t0)
                del m
            out[P.FORMAT_NAMES[f]] = round(float(np.median(ts)) * 1e3, 3)
        except P.PaddingOverflow:
            out[P.FORMAT_NAMES[f]] = "infeasible"
    ts = []
    for r in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        base.extract_features(0.2)
        if r:
            ts.append(time.perf_counter() - t0)
    out["extract_features"] = round(float(np.median(ts)) * 1e3, 3)
    print(name, "ms", json.dumps(out), flush=True)


if __name__ == "__main__":
    bench("laplacian 1000^2", synth.laplacian_2d(1000, seed=1))
    bench("banded 4M x27", synth.banded(4_000_000, 13, seed=2))
    bench("rmat 2^22 d16", synth.rmat(22, 16, seed=42))
