"""Launch list of extract_features and CSR->HDC / CSR->HYB on config 3
(R-MAT 2^22): run under
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ...
(the profiled region is bracketed by cudaProfilerStart/Stop).  Diagnostic."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402

csr = synth.rmat(22, 16, seed=42)
m = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
m.extract_features(0.2)
m.convert(P.HDC)
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.extract_features(0.2)
torch.cuda.synchronize()
m.convert(P.HDC)
torch.cuda.synchronize()
m.convert(P.HYB)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
