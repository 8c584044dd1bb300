import faulthandler, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P
from paper_2303_05098_b200 import synth
faulthandler.dump_traceback_later(40, exit=True)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600_000
csr = synth.hyb_skewed(n, seed=6)
base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
m = base.convert(4)
xd = torch.ones(csr.ncols, dtype=torch.float64, device="cuda"); yd = torch.empty(csr.nrows, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); m.spmv_device(xd.data_ptr(), yd.data_ptr()); torch.cuda.synchronize()
ref = yd.cpu().numpy()
print("device ok", flush=True)
xp = torch.ones(csr.ncols, dtype=torch.float64).pin_memory().numpy(); yp = torch.empty(csr.nrows, dtype=torch.float64).pin_memory().numpy()
for kind in sys.argv[2].split(",") if len(sys.argv) > 2 else ("pinned", "pageable"):
    for i in range(3):
        t0 = time.perf_counter()
        if kind == "pinned":
            m.spmv_into(xp, yp); y = yp
        else:
            y = m.spmv(np.ones(csr.ncols))
        print(kind, i, "%.3f ms" % ((time.perf_counter() - t0) * 1e3), np.array_equal(y, ref), flush=True)
