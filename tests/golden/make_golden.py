"""Generate tests/golden/ref_golden.npz from the REFERENCE itself.

Runs the unmodified reference hot path (compiled in place into
oracle/_ref/libsparseoracle_ref.so by oracle/Makefile) on
  * 40 matrices of the acceptance suite's seeded generator
    (acceptance.cpp:60-66: Rng(1000), random_coo; x from Rng(1001)),
  * three structured instances (2-D Laplacian, banded, R-MAT) at moderate size,
and records SpMV outputs, feature vectors and scan stats per format.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402


def main():
    out = {}
    rng, vrng = O.RefRng(1000), O.RefRng(1001)
    n_mat = 40
    for i in range(n_mat):
        m = rng.random_coo()
        coo = m.export()
        p = f"m{i}_"
        out[p + "nrows"] = coo["nrows"]
        out[p + "ncols"] = coo["ncols"]
        out[p + "row"], out[p + "col"], out[p + "val"] = coo["row"], coo["col"], coo["val"]
        x = vrng.random_vector(coo["ncols"])
        out[p + "x"] = x
        for f in range(6):
            key = f"{p}f{f}_"
            try:
                mf = m.from_coo(f)
            except O.RefError as e:
                assert e.status == 2
                out[key + "feasible"] = 0
                continue
            out[key + "feasible"] = 1
            out[key + "y"] = mf.spmv(x)
            feats, stats = mf.extract_features(0.2)
            out[key + "features"] = feats
            out[key + "stats"] = np.array(stats, np.int64)
    out["n_matrices"] = n_mat

    for name, csr in (("s_lap", synth.laplacian_2d(40, seed=11)),
                      ("s_band", synth.banded(3000, 13, seed=12)),
                      ("s_rmat", synth.rmat(11, 16, seed=13))):
        rows = csr.coo_rows()
        rm = O.RefMatrix.raw_coo(csr.nrows, csr.ncols, rows, csr.col, csr.val).from_coo(O.CSR)
        out[name + "_nrows"], out[name + "_ncols"] = csr.nrows, csr.ncols
        out[name + "_row"], out[name + "_col"], out[name + "_val"] = rows, csr.col, csr.val
        out[name + "_features"] = rm.extract_features(0.2)[0]

    path = os.path.join(HERE, "ref_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
