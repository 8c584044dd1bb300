"""B200 profiling data in the reference's CSV wire formats (wire.py) is read
by the reference's own parsers (ingest.cpp:419-470), joined by its
build_training_csv and trained on by its cmd_train (pipeline.cpp:190-252);
the model it writes loads in the B200 forest loader.  CPU only: the
reference pipeline is compiled in place (oracle/Makefile refpipe)."""
import numpy as np
import pytest

from paper_2303_05098_b200 import forest as F
from paper_2303_05098_b200 import wire as W


def _corpus(O, n=60):
    """Small seeded matrices with oracle features and synthetic per-format
    timings (COO/CSR always feasible; the rest as the oracle's caps say)."""
    rng = O.Rng(2303)
    feats, profs, labels = [], [], []
    for i in range(n):
        coo = rng.random_coo(48)
        row, _ = O.oc_features(O.oc_convert(coo, O.CSR), 0.2)
        mid = f"m{i:03d}"
        feats.append((mid, row))
        best, best_t = None, None
        for f in range(6):
            try:
                O.oc_convert(coo, f)
                feas = True
            except O.PaddingOverflowOracle:
                feas = False
            # a learnable rule: wide rows favour CSR, narrow favour ELL/DIA
            t = (1.0 + 0.1 * f) * (row[5] if f in (2, 3) else row[3] + 2.0) * 1e-6 + 1e-9 * i
            profs.append((mid, f, 50, 50 * t, feas))
            if feas and (best_t is None or 50 * t < best_t):
                best, best_t = f, 50 * t
        labels.append(best)
    return feats, profs, labels


@pytest.fixture(scope="module")
def O():
    import oracle

    if not oracle.refpipe_available():
        pytest.skip("reference pipeline not built (oracle/Makefile refpipe)")
    return oracle


def test_profile_csv_reads_back_exactly(O, tmp_path):
    feats, profs, _ = _corpus(O, 12)
    W.write_profile_csv(tmp_path / "p.csv", profs)
    got = O.ref_read_profile_csv(tmp_path / "p.csv")
    want = [(f, r, t if ok else 0.0, ok) for _, f, r, t, ok in profs]
    assert got == want  # shortest round-trip text: totals are bit-exact


def test_training_join_and_reference_trainer(O, tmp_path):
    feats, profs, labels = _corpus(O)
    W.write_feature_csv(tmp_path / "f.csv", feats)
    W.write_profile_csv(tmp_path / "p.csv", profs)
    written, skipped = O.ref_build_training_csv(tmp_path / "f.csv", tmp_path / "p.csv", tmp_path / "t.csv")
    assert (written, skipped) == (len(feats), 0)
    # build_training_csv labels by the fastest feasible format
    body = (tmp_path / "t.csv").read_text().strip().splitlines()[1:]
    assert [int(line.split(",")[-1]) for line in body] == labels
    rep = O.ref_cmd_train(tmp_path / "f.csv", tmp_path / "p.csv", tmp_path / "model.txt", seed=5, folds=3)
    assert rep["n_train"] + rep["n_test"] == len(feats)
    ff = F.load_model(tmp_path / "model.txt")  # the B200 loader reads the reference's model
    X = np.array([r for _, r in feats])
    pred = F.predict_rows_host(ff, X)
    want = np.array([O.oc_predict_forest(ff, r) for r in X])
    assert np.array_equal(pred, want)
    assert (pred == np.array(labels)).mean() >= 0.6
