"""e2e probe: spmv(m, x) with pinned host buffers on the config-2 matrix
(HDC -> DIA kernel), wall time per call; plus raw H2D / D2H copy rates."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P
from paper_2303_05098_b200 import synth

csr = synth.banded(4_000_000, 13, seed=2)
m = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val).convert(P.HDC)
xh = torch.ones(csr.ncols, dtype=torch.float64).pin_memory(); yh = torch.empty(csr.nrows, dtype=torch.float64).pin_memory()
xn, yn = xh.numpy(), yh.numpy()
for _ in range(5): m.spmv_into(xn, yn)
ts = []
for _ in range(50):
    t0 = time.perf_counter(); m.spmv_into(xn, yn); ts.append(time.perf_counter() - t0)
print("chunks", os.environ.get("SOB_PIPE_CHUNKS", "16"), "e2e ms mean %.3f min %.3f  GB/s %.0f" % (np.mean(ts) * 1e3, np.min(ts) * 1e3, m.spmv_bytes / np.mean(ts) / 1e9))
if os.environ.get("COPY_PROBE"):
    xd = torch.empty_like(xh, device="cuda"); torch.cuda.synchronize()
    for name, f in (("h2d", lambda: xd.copy_(xh, non_blocking=True)), ("d2h", lambda: yh.copy_(xd, non_blocking=True))):
        for _ in range(3): f()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(20): f()
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 20
        print(name, "%.3f ms %.1f GB/s" % (dt * 1e3, 32e6 / dt / 1e9))

if os.environ.get("DUPLEX_PROBE"):
    # full-duplex check: 32 MB H2D and 32 MB D2H on two streams at once
    xd = torch.empty(csr.ncols, dtype=torch.float64, device="cuda")
    yd = torch.empty(csr.nrows, dtype=torch.float64, device="cuda")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(sa):
            xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(sb):
            yh.copy_(yd, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        with torch.cuda.stream(sa):
            xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(sb):
            yh.copy_(yd, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    print("duplex h2d+d2h 2x32MB: %.3f ms, %.1f GB/s aggregate" % (dt * 1e3, 64e6 / dt / 1e9))
    # chunked ping-pong: 16 x 2 MB each way, alternating
    t0 = time.perf_counter()
    for _ in range(20):
        for k in range(16):
            lo, hi = k * csr.nrows // 16, (k + 1) * csr.nrows // 16
            with torch.cuda.stream(sa):
                xd[lo:hi].copy_(xh[lo:hi], non_blocking=True)
            with torch.cuda.stream(sb):
                yh[lo:hi].copy_(yd[lo:hi], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    print("duplex chunked 16x(2+2)MB: %.3f ms, %.1f GB/s aggregate" % (dt * 1e3, 64e6 / dt / 1e9))
