"""Feature-extraction time on arrow matrices (a dense row far past the long-row
cap): the entry-parallel sweep leaves rows of more than 8 SpMV
pieces to piece_sweep.  Prints device time of extract_features (median of 9,
CUDA events inside tune_ml's graph) beside the CSR SpMV time."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402
from paper_2303_05098_b200.models import default_forest  # noqa: E402

forest = P.DeviceForest(default_forest())
for n, dense in ((200_000, 200_000), (1_000_000, 1_000_000), (1_500_000, 300_000)):
    rng = np.random.default_rng(n)
    cols = np.sort(rng.choice(n, dense, replace=False))
    rows = np.concatenate([np.arange(n), np.full(dense, 7)])
    c = np.concatenate([np.arange(n), cols])
    key = np.unique(rows * n + c)
    r, c = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    np.cumsum(rp, out=rp)
    m = P.DeviceMatrix.csr(n, n, rp, c, rng.uniform(0.5, 2, c.size))
    outs = [P.tune_ml(m, forest) for _ in range(10)][1:]
    fe = float(np.median([o.feature_time_seconds for o in outs]))
    per, _ = m.time_spmv(np.ones(n), 20)
    print(f"arrow n={n} dense_row={dense}: T_FE {fe * 1e6:.1f} us, CSR SpMV {np.median(per) * 1e6:.1f} us, "
          f"ratio {fe / np.median(per):.2f}", flush=True)
