#!/usr/bin/env python3
"""Time the device feature pipeline (extract_features and the fused tune_ml)
on chosen config-4 corpus matrices, next to one CSR multiply of the same
matrix.  Run under `ncu --metrics gpu__time_duration.sum` to see which kernel
of the pipeline dominates.

    python scripts/profile_features.py --ids 877 543 --reps 5
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth_dev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ids", type=int, nargs="+", required=True)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--model", default="paper_2303_05098_b200/models/b200_forest.txt")
    a = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    from paper_2303_05098_b200 import forest as F
    forest = P.DeviceForest(F.load_model(a.model))
    for i in a.ids:
        s = synth_dev.corpus_spec(i)
        m = synth_dev.build(s).to_device_matrix()
        fv = m.extract_features(0.2)
        x = torch.ones(fv.ncols, dtype=torch.float64, device="cuda")
        y = torch.empty(fv.nrows, dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
        e0.record(stream)
        for _ in range(a.reps):
            m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        t_csr = e0.elapsed_time(e1) / a.reps
        fe = []
        for _ in range(a.reps):
            e0.record(stream)
            m.extract_features(0.2)
            e1.record(stream)
            e1.synchronize()
            fe.append(e0.elapsed_time(e1))
        P.tune_ml(m, forest)
        outs = [P.tune_ml(m, forest) for _ in range(a.reps)]
        t_fe = np.median([o.feature_time_seconds for o in outs]) * 1e3
        print(f"id {i} {s['family']} n={fv.nrows} nnz={fv.nnz} max_row={fv.to_row()[5]:.0f}: "
              f"csr {t_csr:.3f} ms, extract_features {np.median(fe):.3f} ms, tune t_fe {t_fe:.3f} ms "
              f"({t_fe / t_csr:.1f} CSR-SpMV)", flush=True)


if __name__ == "__main__":
    main()
