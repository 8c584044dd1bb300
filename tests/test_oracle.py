"""CPU: pin the oracle (oracle/oracle.c) before trusting it.

(a) the known-answer tests of the reference's own suites
    (proj/tests/test_formats.cpp, test_spmv.cpp, test_features.cpp,
    test_model.cpp, test_tuners.cpp), restated against the C oracle;
(b) the committed golden fixtures produced by the reference itself
    (tests/golden/make_golden.py -> ref_golden.npz);
(c) when oracle/_ref is present, bit-for-bit agreement with the compiled
    reference on the reference suites' seeded matrices.
"""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ref_golden.npz")

A_TRIPLETS = ([0, 0, 1, 2, 2], [0, 2, 1, 0, 2], [1.0, 2.0, 3.0, 4.0, 5.0])


def worked(O):
    return O.from_triplets(3, 3, *A_TRIPLETS)


def band(O, n, half):  # oracles.hpp:207-217
    r, c, v = [], [], []
    for i in range(n):
        for off in range(-half, half + 1):
            j = i + off
            if 0 <= j < n:
                r.append(i)
                c.append(j)
                v.append(1.0 + float((i + j) % 7))
    return O.from_triplets(n, n, r, c, v)


# ------------------------------------------------------------ formats KATs

def test_canonicalization_sorts_and_sums(O):  # test_formats.cpp:10-21
    m = O.from_triplets(2, 2, [1, 0, 1, 0], [1, 0, 1, 1], [4.0, 1.0, 2.0, 3.0])
    assert m["row"].tolist() == [0, 0, 1]
    assert m["col"].tolist() == [0, 1, 1]
    assert m["val"].tolist() == [1.0, 3.0, 6.0]
    with pytest.raises(O.RefError):
        O.from_triplets(2, 2, [2], [0], [1.0])


def test_rejects_non_canonical(O):  # test_formats.cpp:23-31
    bad = O.coo_dict(2, 2, [1, 0], [0, 0], [1.0, 2.0])
    with pytest.raises(O.RefError):
        O.oc_convert(bad, O.CSR)


def test_worked_example_csr_dia_ell(O):  # test_formats.cpp:33-75
    a = worked(O)
    csr = O.oc_convert(a, O.CSR)
    assert csr["row_ptr"].tolist() == [0, 2, 3, 5]
    assert csr["col"].tolist() == [0, 2, 1, 0, 2]
    assert csr["val"].tolist() == [1, 2, 3, 4, 5]
    dia = O.oc_convert(a, O.DIA)
    assert dia["offsets"].tolist() == [-2, 0, 2]
    assert dia["values"][3:6].tolist() == [1.0, 3.0, 5.0]
    assert dia["values"][0] == 0.0 and dia["values"][1] == 0.0
    ell = O.oc_convert(a, O.ELL)
    assert ell["width"] == 2 and ell["col"][3] == -1


def test_hyb_kh1_and_effective_kh(O):  # test_formats.cpp:98-116
    h = O.oc_convert(worked(O), O.HYB, {"kh_override": 1})
    assert h["ell"]["stored_nnz"] == 3 and h["coo"]["val"].size == 2
    L = O.oc()
    assert L.oc_effective_kh(0, 5, 3) == 2
    assert L.oc_effective_kh(0, 9, 3) == 3
    assert L.oc_effective_kh(0, 0, 3) == 0
    assert L.oc_effective_kh(4, 5, 3) == 4


def test_caps(O):  # test_formats.cpp:118-141
    with pytest.raises(O.PaddingOverflowOracle):
        O.oc_convert(band(O, 100, 1), O.ELL, {"max_padded_entries": 10})
    r = [k % 8 for k in range(40)]
    c = [(k * 7 + k % 8) % 64 for k in range(40)]
    scattered = O.from_triplets(64, 64, r, c, [1.0] * 40)
    with pytest.raises(O.PaddingOverflowOracle):
        O.oc_convert(scattered, O.DIA)


def test_explicit_zeros_kept_in_row_formats(O):  # test_formats.cpp:143-152
    m = O.from_triplets(2, 2, [0, 0, 1], [0, 1, 0], [0.0, 2.0, 3.0])
    assert m["val"].size == 3
    assert O.oc_convert(m, O.CSR)["val"].tolist() == [0.0, 2.0, 3.0]
    e = O.oc_convert(m, O.ELL)
    assert e["col"].tolist() == [0, 1, 0, -1]
    d = O.oc_convert(m, O.DIA)
    assert d["stored_nnz"] == 2  # DIA drops the explicit zero (formats.cpp:93)


# --------------------------------------------------------------- SpMV KATs

def test_spmv_worked_example_all_formats(O):  # test_spmv.cpp:10-18
    a = worked(O)
    for f in range(6):
        assert O.oc_spmv(O.oc_convert(a, f), np.ones(3)).tolist() == [3.0, 3.0, 9.0]


def test_spmv_identity_and_empty(O):  # test_spmv.cpp:20-35
    ident = O.from_triplets(4, 4, range(4), range(4), [1.0] * 4)
    assert O.oc_spmv(O.oc_convert(ident, O.CSR), [1, 2, 3, 4]).tolist() == [1, 2, 3, 4]
    empty = O.coo_dict(3, 3, [], [], [])
    for f in range(6):
        assert O.oc_spmv(O.oc_convert(empty, f), [5, 6, 7]).tolist() == [0, 0, 0]


def test_ell_padding_poison(O):  # test_spmv.cpp:139-150
    e = O.oc_convert(worked(O), O.ELL)
    before = O.oc_spmv(e, np.ones(3))
    e["val"][e["col"] == -1] = 1e9
    assert np.array_equal(O.oc_spmv(e, np.ones(3)), before)


# ----------------------------------------------------------- features KATs

def test_features_worked_example(O):  # test_features.cpp:27-41
    f, _ = O.oc_features(worked(O), 0.5)
    want = [3, 3, 5, 5 / 3, 5 / 9, 2, 1, 2 / 9, 3, 1]
    assert np.allclose(f, want, rtol=1e-12, atol=0)
    assert f[0] == 3 and f[2] == 5 and f[8] == 3 and f[9] == 1


def test_features_identity_and_dense_row(O):  # test_features.cpp:43-72
    for n in (1, 3, 17):
        f, _ = O.oc_features(O.from_triplets(n, n, range(n), range(n), [1.0] * n), 0.2)
        assert f.tolist()[:3] == [n, n, n] and f[3] == 1.0 and f[7] == 0.0
        assert f[8] == 1 and f[9] == 1
    row = O.from_triplets(4, 4, [0] * 4, range(4), [1.0] * 4)
    f, _ = O.oc_features(row, 0.5)
    assert f[5] == 4 and f[6] == 0 and f[8] == 4 and f[9] == 0


def test_features_errors(O):  # test_features.cpp:74-88
    with pytest.raises(O.RefError):
        O.oc_features(O.coo_dict(0, 5, [], [], []), 0.2)
    for bad in (0.0, 1.5):
        with pytest.raises(O.RefError):
            O.oc_features(worked(O), bad)


# -------------------------------------------------------------- model KATs

class _FF:
    def __init__(self, trees, kind=1):
        off, fe, th, le, ri, cl = [0], [], [], [], [], []
        for t in trees:
            for (f, thr, l, r, c) in t:
                fe.append(f)
                th.append(thr)
                le.append(l)
                ri.append(r)
                cl.append(c)
            off.append(off[-1] + len(t))
        self.kind = kind
        self.node_off = np.array(off, np.int64)
        self.feature = np.array(fe, np.int32)
        self.threshold = np.array(th, np.float64)
        self.left = np.array(le, np.int32)
        self.right = np.array(ri, np.int32)
        self.cls = np.array(cl, np.int32)
        self.counts = None


STUMP = [(2, 4.0, 1, 2, -1), (-1, 0.0, -1, -1, 1), (-1, 0.0, -1, -1, 0)]


def test_stump_and_vote_tie(O):  # test_model.cpp:72-118
    ff = _FF([STUMP])
    for nnz, want in ((5, 0), (4, 1), (3, 1)):
        row = np.zeros(10)
        row[:3] = [8, 8, nnz]
        assert O.oc_predict_forest(ff, row) == want
    coo_leaf = [(-1, 0.0, -1, -1, 0)]
    csr_leaf = [(-1, 0.0, -1, -1, 1)]
    assert O.oc_predict_forest(_FF([csr_leaf, csr_leaf, coo_leaf]), np.zeros(10)) == 1
    assert O.oc_predict_forest(_FF([coo_leaf, csr_leaf]), np.zeros(10)) == 0


def test_depth2_tree(O):  # test_model.cpp:80-103
    t = [(2, 10.0, 1, 4, -1), (8, 3.0, 2, 3, -1), (-1, 0, -1, -1, 0), (-1, 0, -1, -1, 1),
         (8, 5.0, 5, 6, -1), (-1, 0, -1, -1, 2), (-1, 0, -1, -1, 3)]
    ff = _FF([t])
    for nnz in (5.0, 15.0):
        for nd in (1.0, 4.0, 7.0):
            row = np.zeros(10)
            row[2], row[8] = nnz, nd
            want = (0 if nd <= 3 else 1) if nnz <= 10 else (2 if nd <= 5 else 3)
            assert O.oc_predict_forest(ff, row) == want


def test_format_feasible_mirrors_conversion(O):  # test_tuners.cpp:297-317
    rng = O.Rng(59)
    for _ in range(100):
        coo = rng.random_coo(48)
        f, _ = O.oc_features(coo, 0.2)
        for t in range(6):
            try:
                O.oc_convert(coo, t)
                actual = True
            except O.PaddingOverflowOracle:
                actual = False
            assert O.oc_format_feasible(t, f) == actual


# ------------------------------------------------------- golden fixtures

@pytest.mark.skipif(not os.path.exists(GOLDEN), reason="golden fixtures not generated")
def test_golden_fixtures(O):
    g = np.load(GOLDEN)
    n_mat = int(g["n_matrices"])
    for i in range(n_mat):
        p = f"m{i}_"
        coo = O.coo_dict(int(g[p + "nrows"]), int(g[p + "ncols"]), g[p + "row"], g[p + "col"], g[p + "val"])
        x = g[p + "x"]
        for f in range(6):
            key = f"{p}f{f}_"
            if int(g[key + "feasible"]) == 0:
                with pytest.raises(O.PaddingOverflowOracle):
                    O.oc_convert(coo, f)
                continue
            m = O.oc_convert(coo, f)
            assert np.array_equal(O.oc_spmv(m, x), g[key + "y"]), (i, f)
            feats, stats = O.oc_features(m, 0.2)
            assert np.array_equal(feats, g[key + "features"]), (i, f)
            assert list(stats) == g[key + "stats"].tolist()
    # structured instances at moderate size (spread parity needs real lengths)
    for name in [k[:-len("_nrows")] for k in g.files if k.startswith("s_") and k.endswith("_nrows")]:
        coo = O.coo_dict(int(g[name + "_nrows"]), int(g[name + "_ncols"]), g[name + "_row"],
                         g[name + "_col"], g[name + "_val"])
        feats, _ = O.oc_features(O.oc_convert(coo, O.CSR), 0.2)
        assert np.array_equal(feats, g[name + "_features"]), name


# --------------------------------------------- live reference (oracle/_ref)

def _cmp(a, b, path=""):
    if isinstance(a, dict):
        for k in a:
            if k != "format":
                _cmp(a[k], b[k], path + "/" + k)
    elif isinstance(a, np.ndarray):
        assert a.dtype == b.dtype and np.array_equal(a, b), path
    else:
        assert a == b, (path, a, b)


def test_oracle_matches_reference_bit_for_bit(O):
    if not O.ref_available():
        try:
            O.build()
        except Exception:
            pytest.skip("reference sources unavailable and no prebuilt oracle/_ref")
    r1, r2, rv = O.Rng(2024), O.RefRng(2024), O.Rng(7)
    feasible = 0
    for t in range(120):
        a = r1.random_coo()
        _cmp(a, r2.random_coo().export())
        for f in range(6):
            try:
                oa = O.oc_convert(a, f)
            except O.PaddingOverflowOracle:
                oa = None
            try:
                rm = O.RefMatrix.from_coo_dict(a).from_coo(f)
            except O.RefError as e:
                assert e.status == 2
                rm = None
            assert (oa is None) == (rm is None), (t, f)
            if oa is None:
                continue
            feasible += 1
            _cmp(oa, rm.export())
            x = rv.random_vector(a["ncols"])
            assert np.array_equal(O.oc_spmv(oa, x), rm.spmv(x)), (t, f)
            for ratio in (0.2, 0.5):
                fo, so_ = O.oc_features(oa, ratio)
                fr, sr = rm.extract_features(ratio)
                assert np.array_equal(fo, fr) and so_ == sr, (t, f)
    assert feasible > 400  # test_formats.cpp:185 expects most targets feasible
