import sys, time, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2303_05098_b200 as P
from paper_2303_05098_b200 import synth
csr = synth.banded(4_000_000, 13, seed=2)
m = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val).convert(P.DIA)
x = np.ones(csr.ncols); y = np.empty(csr.nrows)
for i in range(5): m.spmv_into(x, y)
print("numpy reuse", file=sys.stderr)
for i in range(4): m.spmv_into(x, y)
print("numpy fresh y", file=sys.stderr)
for i in range(4): m.spmv_into(x, np.empty(csr.nrows))
