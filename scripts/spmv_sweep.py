"""Per-format SpMV GB/s on configs 1-3 (device-resident, cold inputs: small
matrices rotate over enough copies to exceed 3x L2, CUDA events on the
launching stream, steps enqueued back to back).  Diagnostic; bench.py carries
the same table for configs 1 and 3 in "other_configs"."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0


def sweep(name, csr, reps=20):
    base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    x = torch.rand(csr.ncols, dtype=torch.float64, device="cuda")
    y = torch.empty(csr.nrows, dtype=torch.float64, device="cuda")
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    out = {}
    for f in range(6):
        try:
            m = base.convert(f)
        except P.PaddingOverflow:
            out[P.FORMAT_NAMES[f]] = "infeasible"
            continue
        ncopy = int(np.ceil(3 * l2 / m.spmv_bytes)) + 1 if m.spmv_bytes < 4 * l2 else 1
        mats = [m] + [m.convert(f) for _ in range(ncopy - 1)]
        xs = [x] + [x.clone() for _ in range(ncopy - 1)]
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps + 3)]
        for k in range(ncopy):  # first multiply of each copy (may profile it), untimed
            mats[k].spmv_device(xs[k].data_ptr(), y.data_ptr(), st.cuda_stream)
        torch.cuda.synchronize()
        for r, (a, b) in enumerate(ev):
            a.record(st)
            mats[r % ncopy].spmv_device(xs[r % ncopy].data_ptr(), y.data_ptr(), st.cuda_stream)
            b.record(st)
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) * 1e-3 for a, b in ev[3:]]
        del mats, xs
        t = float(np.mean(ts))
        nb = m.spmv_bytes
        out[P.FORMAT_NAMES[f]] = f"{t*1e6:8.1f}us {nb/t/1e9:7.0f}GB/s {nb/t/1e9/PEAK:5.3f}"
    print(name, json.dumps(out, indent=1), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["lap", "band", "rmat"]
    if "lap" in which:
        sweep("laplacian 1000^2", synth.laplacian_2d(1000, seed=1))
    if "band" in which:
        sweep("banded 4M x27", synth.banded(4_000_000, 13, seed=2))
    if "rmat" in which:
        sweep("rmat 2^22 d16", synth.rmat(22, 16, seed=42))
