"""Host-buffer spmv(m, x) per format on config 2 (banded 4M x 27) and the
HYB-shaped matrix (4M, 16/160-entry rows): wall ms per call with pinned and
pageable x/y.  Measurement script for the A/B recipes (scripts/gpu_r02*.sh).

    python scripts/e2e_formats.py [formats, default 0,4]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402

fmts = [int(f) for f in (sys.argv[1] if len(sys.argv) > 1 else "0,4").split(",")]
for name, csr in (("banded", synth.banded(4_000_000, 13, seed=2)), ("hyb", synth.hyb_skewed(4_000_000, seed=6))):
    base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    x = np.ones(csr.ncols)
    y = np.empty(csr.nrows)
    xp = torch.ones(csr.ncols, dtype=torch.float64).pin_memory().numpy()
    yp = torch.empty(csr.nrows, dtype=torch.float64).pin_memory().numpy()
    for f in fmts:
        try:
            m = base.convert(f)
        except P.PaddingOverflow:
            print(name, f, "infeasible", flush=True)
            continue
        for kind, (xx, yy) in (("pageable", (x, y)), ("pinned", (xp, yp))):
            for _ in range(3):
                m.spmv_into(xx, yy)
            ts = []
            for _ in range(20):
                t0 = time.perf_counter()
                m.spmv_into(xx, yy)
                ts.append(time.perf_counter() - t0)
            print(name, f, kind, "ms mean %.3f min %.3f" % (np.mean(ts) * 1e3, np.min(ts) * 1e3), flush=True)
