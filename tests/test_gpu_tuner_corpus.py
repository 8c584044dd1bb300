"""GPU parity of the fused tuner on real forests and of the config-4 corpus.

* The single-row predict path of ``so_tune_ml`` (blocked layout, warp walk
  across depth-5 blocks, model.cu ``walk_warp2``) against the oracle's
  ``predict_forest`` (model.cpp:215-228) for the shipped forests, a
  reference-trained forest and a synthetic 100-tree depth-16 forest, on 10K+
  feature rows: random rows, rows sitting exactly on split thresholds
  (``x <= thr`` goes left, model.cpp:206-209), the 400 held-out config-4 rows
  and vote ties (ties -> lowest FormatId).
* ``tune_ml`` end to end (features -> predict -> format_feasible -> CSR
  fallback, tuners.cpp:92-114) with those forests on seeded matrices.
* ~100 matrices of the config-4 corpus (all four families, up to the largest
  5M-row power-law ones), device-generated: all ten features bit-exact
  against the oracle's extract_features (features.cpp:82-153) and the tuned
  label equal to the oracle's prediction + feasibility.
"""
import csv
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODELS = os.path.join(REPO, "paper_2303_05098_b200", "models")


def _load(name):
    from paper_2303_05098_b200 import forest as F
    return F.load_model(os.path.join(MODELS, name))


def synthetic_deep_forest(n_trees=100, depth=16, seed=7, kind=1):
    """Random trees reaching `depth` (a guaranteed spine per tree), splits on
    every feature with thresholds drawn from the row distribution below."""
    from paper_2303_05098_b200.device import FlatForest
    rng = np.random.default_rng(seed)
    off, fe, th, le, ri, cl = [0], [], [], [], [], []
    for t in range(n_trees):
        nodes = []  # (feature, thr, left, right, cls)

        def grow(d, spine):
            idx = len(nodes)
            nodes.append(None)
            split = d < depth and (spine or d < 3 or rng.random() < 0.72)
            if not split:
                nodes[idx] = (-1, 0.0, -1, -1, int(rng.integers(6)))
                return idx
            f = int(rng.integers(10))
            thr = float(_feature_value(rng, f))
            go_left = bool(rng.integers(2))
            l = grow(d + 1, spine and go_left)
            r = grow(d + 1, spine and not go_left)
            nodes[idx] = (f, thr, l, r, -1)
            return idx

        grow(0, True)
        for f, tv, l, r, c in nodes:
            fe.append(f), th.append(tv), le.append(l), ri.append(r), cl.append(c)
        off.append(len(fe))
    return FlatForest(kind, np.array(off, np.int64), np.array(fe, np.int32), np.array(th, np.float64),
                      np.array(le, np.int32), np.array(ri, np.int32), np.array(cl, np.int32))


def _feature_value(rng, f):
    """A plausible value of feature f (features_to_row order)."""
    n = float(np.exp(rng.uniform(np.log(1e3), np.log(1e8))))
    return {0: round(n), 1: round(n), 2: round(n * rng.uniform(1, 40)), 3: rng.uniform(1, 40),
            4: 10 ** rng.uniform(-8, -1), 5: float(rng.integers(1, 5000)), 6: float(rng.integers(0, 30)),
            7: 10 ** rng.uniform(-3, 5), 8: float(rng.integers(1, 2_000_000)),
            9: float(rng.integers(0, 200))}[f]


def feature_rows(ff, count, seed):
    """Random rows, plus rows whose features equal split thresholds exactly."""
    rng = np.random.default_rng(seed)
    rows = np.array([[_feature_value(rng, f) for f in range(10)] for _ in range(count)])
    split = np.flatnonzero(ff.feature >= 0)
    pick = rng.choice(split, size=min(count // 2, split.size), replace=split.size < count // 2)
    for k, node in enumerate(pick):
        rows[k, ff.feature[node]] = ff.threshold[node]  # x == thr -> left
    return rows


def held_out_rows():
    path = os.path.join(REPO, "profiles", "config4_tuned_r01e.csv")
    with open(path) as f:
        return np.array([[float(r[f"f{k}"]) for k in range(10)] for r in csv.DictReader(f)])


def first_tree(ff):
    from paper_2303_05098_b200.device import FlatForest
    e = int(ff.node_off[1])
    return FlatForest(0, ff.node_off[:2].copy(), ff.feature[:e], ff.threshold[:e], ff.left[:e], ff.right[:e],
                      ff.cls[:e])


FORESTS = {
    "b200_forest": lambda: _load("b200_forest.txt"),
    "b200_forest_reftrained": lambda: _load("b200_forest_reftrained.txt"),
    "b200_tree": lambda: _load("b200_forest_tree.txt"),
    "synthetic_100x16": lambda: synthetic_deep_forest(),
}


@pytest.mark.parametrize("name", sorted(FORESTS))
def test_latency_predict_matches_oracle(so, O, name):
    ff = FORESTS[name]()
    rows = np.concatenate([feature_rows(ff, 10_000, seed=len(name)), held_out_rows()])
    df = so.DeviceForest(ff)
    # a tree model predicts with trees.front() (tuners.cpp:103-105); a forest votes over all
    want_ff = first_tree(ff) if ff.kind == 0 else ff
    want = np.array([O.oc_predict_forest(want_ff, r) for r in rows], np.int32)
    assert np.array_equal(df.predict_rows_latency(rows), want)
    if ff.kind == 1:
        assert np.array_equal(df.predict_rows(rows), want)  # throughput path agrees
    # the C++ predict entry (so_predict) runs the same latency path
    for r in rows[:64]:
        assert df.predict(so.FeatureVector.from_row(list(r))) == O.oc_predict_forest(want_ff, r)


def test_vote_ties_go_to_lowest_id(so, O):
    """Forests whose votes tie between classes: argmax with strict '>'."""
    from paper_2303_05098_b200.device import FlatForest
    rng = np.random.default_rng(3)
    trees = []
    for _ in range(12):  # stumps on nnz, random leaf classes: many rows tie 2-2-2 etc.
        thr = float(rng.integers(10, 1000))
        trees.append([(2, thr, 1, 2, -1), (-1, 0.0, -1, -1, int(rng.integers(6))),
                      (-1, 0.0, -1, -1, int(rng.integers(6)))])
    off, fe, th, le, ri, cl = [0], [], [], [], [], []
    for t in trees:
        for f, tv, l, r, c in t:
            fe.append(f), th.append(tv), le.append(l), ri.append(r), cl.append(c)
        off.append(len(fe))
    ff = FlatForest(1, np.array(off, np.int64), np.array(fe, np.int32), np.array(th, np.float64),
                    np.array(le, np.int32), np.array(ri, np.int32), np.array(cl, np.int32))
    rows = np.zeros((2000, 10))
    rows[:, 2] = rng.integers(0, 1100, 2000)
    want = np.array([O.oc_predict_forest(ff, r) for r in rows], np.int32)
    assert np.array_equal(so.DeviceForest(ff).predict_rows_latency(rows), want)


def _oracle_tune(O, ff, fo, cfg=None):
    want_ff = first_tree(ff) if ff.kind == 0 else ff
    p = O.oc_predict_forest(want_ff, fo)
    if not O.oc_format_feasible(p, fo, cfg):
        return 1, 1
    return p, 0


@pytest.mark.parametrize("name", sorted(FORESTS))
def test_tune_ml_real_forests_vs_oracle(so, O, name):
    """tune_ml end to end on seeded matrices of every format."""
    from paper_2303_05098_b200 import synth
    ff = FORESTS[name]()
    df = so.DeviceForest(ff)
    rng = O.Rng(77)
    mats = [rng.random_coo(int(rng.uniform_index(200)) + 2) for _ in range(60)]
    for csr in (synth.banded(30_000, 5, seed=2), synth.rmat(14, 12, seed=3), synth.laplacian_2d(120, seed=1),
                synth.uniform_random(40_000, 9, seed=4), synth.hyb_skewed(30_000, 6, 90, 17, seed=8)):
        mats.append(O.coo_dict(csr.nrows, csr.ncols, csr.coo_rows(), csr.col, csr.val))
    for k, coo in enumerate(mats):
        fo, _ = O.oc_features(O.oc_convert(coo, O.CSR), 0.2)
        chosen, fb = _oracle_tune(O, ff, fo)
        d = so.DeviceMatrix.coo(coo["nrows"], coo["ncols"], coo["row"], coo["col"], coo["val"])
        for fmt in (k % 6, 1):
            try:
                m = d.from_coo(fmt)
            except so.PaddingOverflow:
                continue
            o = so.tune_ml(m, df)
            assert o.features.to_row() == fo.tolist(), (k, fmt)
            assert (o.chosen, o.fallback_csr) == (chosen, fb), (k, fmt)
            assert o.switched == int(chosen != fmt)
            assert o.source == (1 if ff.kind == 0 else 2)


def _corpus_ids(per_family=25, nmax=5_000_000):
    """~per_family ids per family spread over the size range, plus the
    largest power-law matrices of the 2000-matrix batch."""
    from paper_2303_05098_b200 import synth_dev
    specs = [synth_dev.corpus_spec(i, nmax=nmax) for i in range(2000)]
    ids = []
    for fam in synth_dev.FAMILIES:
        fs = sorted((s for s in specs if s["family"] == fam), key=lambda s: synth_dev.nnz_estimate(s))
        pick = np.unique(np.linspace(0, len(fs) - 1, per_family).round().astype(int))
        ids += [fs[p]["id"] for p in pick]
    pl = sorted((s for s in specs if s["family"] == "powerlaw"), key=lambda s: -s["n"])
    ids += [s["id"] for s in pl[:3]]
    return sorted(set(ids))


def test_corpus_ids_cover_families():
    from paper_2303_05098_b200 import synth_dev
    ids = _corpus_ids()
    fams = {synth_dev.corpus_spec(i)["family"] for i in ids}
    assert fams == set(synth_dev.FAMILIES) and len(ids) >= 90


def test_config4_corpus_features_and_labels(so, O):
    import torch
    from paper_2303_05098_b200 import synth_dev
    forest_ff = _load("b200_forest.txt")
    df = so.DeviceForest(forest_ff)
    checked = {f: 0 for f in synth_dev.FAMILIES}
    largest = 0
    for i in _corpus_ids():
        spec = synth_dev.corpus_spec(i)
        dc = synth_dev.build(spec)
        m = dc.to_device_matrix()
        host = {"format": O.CSR, "nrows": dc.nrows, "ncols": dc.ncols,
                "row_ptr": dc.row_ptr.cpu().numpy().astype(np.int64),
                "col": dc.col.cpu().numpy().astype(np.int64), "val": dc.val.cpu().numpy()}
        del dc
        torch.cuda.empty_cache()
        fo, _ = O.oc_features(host, 0.2)
        fv = m.extract_features(0.2)
        assert np.array_equal(np.array(fv.to_row()), fo), (i, spec["family"], fv.to_row(), fo.tolist())
        o = so.tune_ml(m, df)
        assert o.features.to_row() == fo.tolist(), i
        chosen, fb = _oracle_tune(O, forest_ff, fo)
        assert (o.chosen, o.fallback_csr) == (chosen, fb), (i, spec["family"])
        checked[spec["family"]] += 1
        largest = max(largest, host["nrows"])
        del m, host
    assert all(v >= 20 for v in checked.values()), checked
    assert largest >= 4_000_000
