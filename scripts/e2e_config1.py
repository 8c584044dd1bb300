"""config 1 (2-D Laplacian 1000^2, DIA, offsets +-1000): pinned spmv(m, x) wall time per call."""
import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2303_05098_b200 as P
from paper_2303_05098_b200 import synth
csr = synth.laplacian_2d(1000, seed=1)
m = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val).convert(2)
xp = torch.ones(csr.ncols, dtype=torch.float64).pin_memory().numpy(); yp = torch.empty(csr.nrows, dtype=torch.float64).pin_memory().numpy()
for _ in range(5): m.spmv_into(xp, yp)
ts = []
for _ in range(30):
    t0 = time.perf_counter(); m.spmv_into(xp, yp); ts.append(time.perf_counter() - t0)
print("config1 DIA pinned spmv(m, x) ms median %.3f min %.3f" % (np.median(ts) * 1e3, np.min(ts) * 1e3))
