"""CPU: the C-ABI library and the C++ drop-in load and export their symbols
(no compute calls without a GPU), and the host-side tooling behaves."""
import os
import re
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "sparseoracle_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(so_[a-z0-9_]+)\s*\(", text)))


def exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if ln.strip()}


def test_c_abi_exports_every_declared_symbol():
    from paper_2303_05098_b200 import _capi

    if not os.path.exists(_capi.LIB_PATH):
        _capi.build()
    syms = exported(_capi.LIB_PATH)
    missing = [f for f in declared_functions() if f not in syms]
    assert not missing, missing
    assert len(declared_functions()) >= 25


def test_ctypes_binding_covers_header():
    from paper_2303_05098_b200 import _capi

    assert set(declared_functions()) == set(_capi.exported_symbols())


def test_library_loads_and_fails_loudly_without_gpu():
    import torch

    from paper_2303_05098_b200 import _capi
    import paper_2303_05098_b200 as P

    lib = _capi.lib()
    assert lib.so_version().startswith(b"sparseoracle-b200")
    if not torch.cuda.is_available():
        with pytest.raises(P.Error):  # no silent host path
            P.DeviceMatrix.coo(3, 3, [0], [0], [1.0])


def test_cpp_api_exports_reference_surface():
    lib = os.path.join(REPO, "paper_2303_05098_b200", "lib", "libsparseoracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", REPO, "-j8"], check=True, capture_output=True)
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True).stdout
    for sym in ["sparseoracle::spmv(", "sparseoracle::spmv_parallel(", "sparseoracle::time_spmv(",
                "sparseoracle::from_coo(", "sparseoracle::to_coo(", "sparseoracle::switch_format(",
                "sparseoracle::extract_features(", "sparseoracle::predict_tree(",
                "sparseoracle::predict_forest(", "sparseoracle::load_model(", "sparseoracle::save_model(",
                "sparseoracle::tune_ml(", "sparseoracle::tune_multiply(", "sparseoracle::tune_run_first(",
                "sparseoracle::format_feasible(", "sparseoracle::CooMatrix::from_triplets("]:
        assert sym in out, sym


def test_forest_tooling_roundtrip_and_reference_loader(tmp_path):
    from paper_2303_05098_b200 import forest as F

    rng = np.random.default_rng(0)
    X = rng.uniform(0, 100, (300, 10))
    X[:, [0, 1, 2, 5, 6, 8, 9]] = np.floor(X[:, [0, 1, 2, 5, 6, 8, 9]])  # integer feature fields
    y = (X[:, 2] > 50).astype(int) + 2 * (X[:, 8] > 70).astype(int)
    ff = F.train_forest(X, y, n_estimators=5, max_depth=6, seed=1)
    pred = F.predict_rows_host(ff, X)
    assert (pred == y).mean() > 0.9
    p1, p2 = tmp_path / "a.txt", tmp_path / "b.txt"
    F.save_model(ff, p1, [("backend", "b200")])
    F.save_model(F.load_model(p1), p2, [("backend", "b200")])
    assert p1.read_bytes() == p2.read_bytes()
    import oracle as O
    if O.ref_available() or os.path.isdir("/root/reference/proj"):
        import ctypes as C
        h = C.c_void_p()
        assert O.ref().ref_load_model(str(p1).encode(), C.byref(h)) == 0  # the reference parser accepts it
        rows = X[:50]
        got = [O.ref().ref_predict_forest(h, O._p(np.ascontiguousarray(r))) for r in rows]
        assert got == F.predict_rows_host(ff, rows).tolist()
        O.ref().ref_forest_free(h)


def test_format_double_matches_to_chars():
    from paper_2303_05098_b200.forest import format_double

    cases = {0.1: "0.1", 1 / 3: "0.3333333333333333", 1e300: "1e+300", 4.0: "4", 0.0001: "1e-04",
             123456.0: "123456", 1e16: "1e+16", 1.5e-7: "1.5e-07", 0.5: "0.5", 100.0: "100"}
    for v, want in cases.items():
        assert format_double(v) == want, v


def test_synth_generators_are_canonical():
    from paper_2303_05098_b200 import synth

    for csr in (synth.laplacian_2d(30), synth.banded(500, 4), synth.stencil_3d(8), synth.rmat(10, 8),
                synth.uniform_random(400, 6)):
        rp, col = csr.row_ptr, csr.col
        assert rp[0] == 0 and rp[-1] == csr.nnz and np.all(np.diff(rp) >= 0)
        for r in range(csr.nrows):
            seg = col[rp[r]:rp[r + 1]]
            assert np.all(np.diff(seg) > 0) and (seg.size == 0 or (seg[0] >= 0 and seg[-1] < csr.ncols))
    lap = synth.laplacian_2d(1000)
    assert lap.nnz == 5 * 1000 * 1000 - 4 * 1000  # z = 5n - 4g
    band = synth.banded(4000, 13)
    assert band.nnz == 27 * 4000 - 13 * 14


def test_corpus_spec_mix_and_lpt_sharding():
    import importlib.util

    from paper_2303_05098_b200 import synth_dev

    specs = [synth_dev.corpus_spec(i) for i in range(2000)]
    fams = [s["family"] for s in specs]
    assert all(fams.count(f) == 500 for f in synth_dev.FAMILIES)
    assert all(10_000 <= s["n"] <= 5_000_000 for s in specs)
    spec = importlib.util.spec_from_file_location("config4", os.path.join(REPO, "scripts", "config4.py"))
    c4 = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(c4)
    shards = [c4.lpt_shard(specs[:200], 4, r) for r in range(4)]
    ids = sorted(s["id"] for sh in shards for s in sh)
    assert ids == list(range(200))
    loads = [sum(synth_dev.nnz_estimate(s) for s in sh) for sh in shards]
    assert max(loads) / min(loads) < 1.2
