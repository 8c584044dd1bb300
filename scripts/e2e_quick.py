import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2303_05098_b200 as P
from paper_2303_05098_b200 import synth
csr = synth.banded(4_000_000, 13, seed=2)
base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
for f in (2, 1, 0, 3):
    m = base.convert(f)
    nb = m.spmv_bytes
    x = np.ones(csr.ncols); y = np.empty(csr.nrows)
    xp = torch.ones(csr.ncols, dtype=torch.float64).pin_memory().numpy(); yp = torch.empty(csr.nrows, dtype=torch.float64).pin_memory().numpy()
    for name, (xx, yy) in (("pageable", (x, y)), ("pinned", (xp, yp))):
        for _ in range(3): m.spmv_into(xx, yy)
        ts = []
        for _ in range(20):
            t0 = time.perf_counter(); m.spmv_into(xx, yy); ts.append(time.perf_counter() - t0)
        print(f, name, "ms mean %.3f min %.3f GB/s %.1f" % (np.mean(ts)*1e3, np.min(ts)*1e3, nb/np.mean(ts)/1e9), flush=True)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); yy = m.spmv(x); ts.append(time.perf_counter() - t0)
    print(f, "fresh-y pageable ms %.3f" % (np.mean(ts)*1e3), flush=True)
import os
print("cpus", os.cpu_count())
