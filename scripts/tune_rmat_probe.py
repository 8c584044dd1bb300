#!/usr/bin/env python3
"""tune_ml on the config-3 R-MAT (and config 2) matrices: device T_FE /
T_PRED and host wall of steady-state calls (the first call builds the plan)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if os.environ.get("AB_ROOT"):
    sys.path.insert(0, os.environ["AB_ROOT"])


def main():
    import paper_2303_05098_b200 as P
    from paper_2303_05098_b200 import synth
    forest = P.DeviceForest(bench.forest_ff())
    for name, csr in (("rmat", synth.rmat(22, 16, seed=42)), ("banded", synth.banded(4_000_000, 13, seed=2))):
        d = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
        P.tune_ml(d, forest)
        outs = [P.tune_ml(d, forest) for _ in range(5)]
        fe = np.median([o.feature_time_seconds for o in outs]) * 1e3
        pr = np.median([o.predict_time_seconds for o in outs]) * 1e3
        wa = np.median([o.wall_time_seconds for o in outs]) * 1e3
        print(f"{name} tune_ml T_FE {fe:.3f} ms T_PRED {pr:.4f} ms wall {wa:.3f} ms chosen {P.FORMAT_NAMES[outs[-1].chosen]}",
              flush=True)


if __name__ == "__main__":
    main()
