"""Repro loop for an intermittent stall in test_pageable_host_spmv_staging[wide]
(laplacian_2d(800), pageable 8-byte-aligned x / y, every format): fresh
matrices each round; faulthandler dumps every thread's Python stack and
exits if one round takes longer than 20 s.

    python scripts/pageable_stall_repro.py [rounds]
"""
import faulthandler
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as so  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 100
csr = synth.laplacian_2d(800, seed=1)
rng = np.random.default_rng(12)
t_start = time.time()
for it in range(rounds):
    faulthandler.dump_traceback_later(20, exit=True)
    d = so.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    for f in range(6):
        try:
            m = d.convert(f)
        except so.PaddingOverflow:
            continue
        big = rng.uniform(-1, 1, csr.ncols + 3)
        x = big[1:1 + csr.ncols]
        yb = np.full(csr.nrows + 2, np.nan)
        y = yb[1:1 + csr.nrows]
        print(f"round {it} format {f} spmv_into", file=sys.stderr, flush=True)
        m.spmv_into(x, y)
        xd = torch.tensor(x, device="cuda")
        yd = torch.empty(csr.nrows, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        m.spmv_device(xd.data_ptr(), yd.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(y, yd.cpu().numpy()), (it, f)
        for k in range(2):
            print(f"round {it} format {f} spmv {k}", file=sys.stderr, flush=True)
            assert np.array_equal(m.spmv(x), y), (it, f)
            print(f"round {it} format {f} spmv_new {k}", file=sys.stderr, flush=True)
            assert np.array_equal(m.spmv_new(x), y), (it, f)
    faulthandler.cancel_dump_traceback_later()
print(f"{rounds} rounds clean in {time.time() - t_start:.1f} s")
