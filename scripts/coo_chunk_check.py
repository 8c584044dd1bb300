"""Pinned COO chunk pipeline on config 2 (banded 4M x 27, 108M entries: the
device multiply takes the records + fix-up path, the pinned call the CONT
chunk kernel): max relative difference between the two, and wall ms per
pinned call.  Measurement script for scripts/gpu_r02_coochunks.sh.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402

csr = synth.banded(4_000_000, 13, seed=2)
m = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val).convert(0)
xp = torch.empty(csr.ncols, dtype=torch.float64).pin_memory().numpy()
yp = torch.empty(csr.nrows, dtype=torch.float64).pin_memory().numpy()
xp[:] = np.random.default_rng(3).uniform(-1, 1, csr.ncols)
m.spmv_into(xp, yp)
xd = torch.tensor(xp, device="cuda")
yd = torch.empty(csr.nrows, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
m.spmv_device(xd.data_ptr(), yd.data_ptr())
torch.cuda.synchronize()
ref = yd.cpu().numpy()
rel = np.max(np.abs(yp - ref) / np.maximum(np.abs(ref), 1e-300))
ts = []
for _ in range(30):
    t0 = time.perf_counter()
    m.spmv_into(xp, yp)
    ts.append(time.perf_counter() - t0)
ts = np.array(ts[5:]) * 1e3
print(f"COO pinned ms mean {ts.mean():.3f} min {ts.min():.3f}; max rel vs device {rel:.3e}; "
      f"bitwise {np.array_equal(yp, ref)}; chunks {'off' if os.environ.get('SOB_NO_COO_CHUNKS') else 'on'}")
