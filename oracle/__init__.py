"""TEST INFRASTRUCTURE ONLY -- the parity oracle, never the product.

Python (ctypes) view of
  * ``oracle/_build/liboracle.so`` -- the plain-C restatement (oracle.c), and
  * ``oracle/_ref/libsparseoracle_ref.so`` -- the unmodified reference sources
    compiled in place (oracle/Makefile) behind a tiny extern "C" shim.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
reference arm may import this package.  Host-layout dicts use the same keys as
``paper_2303_05098_b200.DeviceMatrix.download()``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libsparseoracle_ref.so")
# the reference's pipeline / trainer / CSV wire formats (optional, oracle/Makefile refpipe)
REFPIPE_LIB = os.path.join(HERE, "_ref", "libsparseoracle_refpipe.so")

COO, CSR, DIA, ELL, HYB, HDC = range(6)
vp = C.c_void_p
i64 = C.c_int64
f64 = C.c_double

_oc = None
_ref = None


def build():
    subprocess.run(["make", "-C", HERE], check=True, stdout=subprocess.DEVNULL)


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


def oc():
    global _oc
    if _oc is None:
        if not os.path.exists(ORACLE_LIB):
            build()
        _oc = C.CDLL(ORACLE_LIB)
        L = _oc
        L.oc_rng_seed.argtypes = [vp, C.c_uint64]
        L.oc_rng_next.restype = C.c_uint64
        L.oc_rng_next.argtypes = [vp]
        L.oc_rng_uniform_index.restype = C.c_uint64
        L.oc_rng_uniform_index.argtypes = [vp, C.c_uint64]
        L.oc_rng_uniform_real.restype = f64
        L.oc_rng_uniform_real.argtypes = [vp, f64, f64]
        L.oc_derive_seed.restype = C.c_uint64
        L.oc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.oc_random_coo.argtypes = [vp, i64, f64, f64, vp, vp, vp, vp, vp, vp]
        L.oc_random_vector.argtypes = [vp, i64, vp]
        L.oc_from_triplets.argtypes = [i64, i64, i64, vp, vp, vp, vp]
        L.oc_is_canonical.argtypes = [i64, i64, i64, vp, vp]
        L.oc_padded_entry_cap.restype = i64
        L.oc_padded_entry_cap.argtypes = [f64, i64, i64]
        L.oc_effective_kh.restype = i64
        L.oc_effective_kh.argtypes = [i64, i64, i64]
        L.oc_true_diag_threshold.restype = i64
        L.oc_true_diag_threshold.argtypes = [f64, i64, i64]
        L.oc_coo_to_csr.argtypes = [i64, i64, vp, vp]
        L.oc_dia_plan.argtypes = [i64, i64, i64, vp, vp, vp, i64, vp, vp]
        L.oc_dia_fill.argtypes = [i64, i64, i64, vp, vp, vp, vp, i64, vp, vp, vp]
        L.oc_ell_plan.argtypes = [i64, i64, vp, i64, vp]
        L.oc_ell_fill.argtypes = [i64, i64, vp, vp, vp, i64, vp, vp]
        L.oc_hyb_plan.argtypes = [i64, i64, vp, i64, i64, vp, vp]
        L.oc_hyb_fill.argtypes = [i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp]
        L.oc_hdc_plan.argtypes = [i64, i64, i64, vp, vp, i64, i64, vp, vp, vp]
        L.oc_hdc_fill.argtypes = [i64, i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp, vp]
        L.oc_spmv_coo.argtypes = [i64, i64, vp, vp, vp, vp, vp, C.c_int]
        L.oc_spmv_csr.argtypes = [i64, vp, vp, vp, vp, vp, C.c_int]
        L.oc_spmv_dia.argtypes = [i64, i64, i64, vp, vp, vp, vp, C.c_int]
        L.oc_spmv_ell.argtypes = [i64, i64, vp, vp, vp, vp, C.c_int]
        L.oc_extract_features.argtypes = [vp, f64, vp, vp]
        L.oc_predict_tree.argtypes = [vp, vp, vp, vp, vp, vp]
        L.oc_predict_forest.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, vp]
        L.oc_format_feasible.argtypes = [C.c_int, vp, i64, f64, i64]
    return _oc


_refpipe = None


def refpipe_available():
    return os.path.exists(REFPIPE_LIB)


def refpipe():
    """ctypes view of oracle/ref_pipeline_capi.cpp (reference cmd_train,
    read_profile_csv, build_training_csv)."""
    global _refpipe
    if _refpipe is None:
        L = C.CDLL(REFPIPE_LIB)
        L.refp_last_error.restype = C.c_char_p
        L.refp_cmd_train.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint64, C.c_int,
                                     C.POINTER(f64), C.POINTER(f64), C.POINTER(i64), C.POINTER(i64)]
        L.refp_read_profile_csv.argtypes = [C.c_char_p, i64, C.POINTER(i64), C.POINTER(C.c_int32),
                                            C.POINTER(i64), C.POINTER(f64), C.POINTER(C.c_int32)]
        L.refp_build_training_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(i64), C.POINTER(i64)]
        L.refp_read_mm.argtypes = [C.c_char_p, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(C.c_int32)]
        L.refp_mm_arrays.argtypes = [vp, vp, vp]
        L.refp_mm_arrays.restype = None
        L.refp_write_mm.argtypes = [C.c_char_p, i64, i64, i64, vp, vp, vp]
        _refpipe = L
    return _refpipe


def _pchk(L, st):
    if st != 0:
        raise RuntimeError(L.refp_last_error().decode(errors="replace"))


def ref_cmd_train(features_csv, profiles_csv, model_out, seed=0, folds=5):
    """The reference's cmd_train (pipeline.cpp:190-252) on CSV files."""
    L = refpipe()
    acc, bacc, ntr, nte = f64(), f64(), i64(), i64()
    _pchk(L, L.refp_cmd_train(str(features_csv).encode(), str(profiles_csv).encode(), str(model_out).encode(),
                              seed, folds, C.byref(acc), C.byref(bacc), C.byref(ntr), C.byref(nte)))
    return {"heldout_accuracy": acc.value, "heldout_balanced_accuracy": bacc.value,
            "n_train": ntr.value, "n_test": nte.value}


def ref_read_profile_csv(path):
    """[(format, repetitions, total_seconds, feasible)] via the reference reader."""
    L = refpipe()
    cnt, fm, reps, tot, feas = i64(), C.c_int32(), i64(), f64(), C.c_int32()
    _pchk(L, L.refp_read_profile_csv(str(path).encode(), -1, C.byref(cnt), C.byref(fm), C.byref(reps),
                                     C.byref(tot), C.byref(feas)))
    out = []
    for i in range(cnt.value):
        _pchk(L, L.refp_read_profile_csv(str(path).encode(), i, C.byref(cnt), C.byref(fm), C.byref(reps),
                                         C.byref(tot), C.byref(feas)))
        out.append((fm.value, reps.value, tot.value, bool(feas.value)))
    return out


def ref_build_training_csv(features_csv, profiles_csv, out_csv):
    L = refpipe()
    w, sk = i64(), i64()
    _pchk(L, L.refp_build_training_csv(str(features_csv).encode(), str(profiles_csv).encode(),
                                       str(out_csv).encode(), C.byref(w), C.byref(sk)))
    return w.value, sk.value


MM_ERRORS = {1: "ParseError", 2: "UnsupportedFormat", 3: "IndexOutOfRange", 4: "Error"}


def ref_read_matrix_market(path):
    """The reference's read_matrix_market: ('ok', coo dict) or (error type
    name, message)."""
    L = refpipe()
    n, m, z, kind = i64(), i64(), i64(), C.c_int32()
    if L.refp_read_mm(str(path).encode(), C.byref(n), C.byref(m), C.byref(z), C.byref(kind)) != 0:
        return MM_ERRORS[kind.value], L.refp_last_error().decode(errors="replace")
    row, col, val = np.zeros(z.value, np.int64), np.zeros(z.value, np.int64), np.zeros(z.value)
    L.refp_mm_arrays(_p(row), _p(col), _p(val))
    return "ok", {"format": COO, "nrows": n.value, "ncols": m.value, "row": row, "col": col, "val": val}


def ref_write_matrix_market(path, coo):
    L = refpipe()
    row, col, val = (np.ascontiguousarray(coo["row"], np.int64), np.ascontiguousarray(coo["col"], np.int64),
                     np.ascontiguousarray(coo["val"], np.float64))
    _pchk(L, L.refp_write_mm(str(path).encode(), coo["nrows"], coo["ncols"], val.size, _p(row), _p(col), _p(val)))


def ref_available():
    return os.path.exists(REF_LIB)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            build()
        L = C.CDLL(REF_LIB)
        L.ref_last_error.restype = C.c_char_p
        for name, args in {
            "ref_coo_from_triplets": [i64, i64, i64, vp, vp, vp, C.POINTER(vp)],
            "ref_coo_raw": [i64, i64, i64, vp, vp, vp, C.POINTER(vp)],
            "ref_clone": [vp, C.POINTER(vp)],
            "ref_from_coo": [vp, C.c_int, i64, f64, f64, i64, C.POINTER(vp)],
            "ref_switch_format": [vp, C.c_int, i64, f64, f64, i64],
            "ref_to_coo": [vp, C.POINTER(vp)],
            "ref_spmv": [vp, vp, i64, vp, C.c_int],
            "ref_time_spmv": [vp, vp, i64, i64, C.c_int, vp, vp],
            "ref_extract_features": [vp, f64, vp, vp],
            "ref_forest_create": [C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp, C.POINTER(vp)],
            "ref_load_model": [C.c_char_p, C.POINTER(vp)],
            "ref_save_model": [vp, C.c_char_p],
            "ref_tune_ml": [vp, vp, f64, i64, f64, i64, vp, vp],
            "ref_tune_multiply": [vp, vp, i64, C.c_int, vp, i64, C.c_int, vp, vp],
            "ref_random_coo": [vp, i64, f64, f64, C.POINTER(vp)],
            "ref_band_matrix": [i64, i64, C.POINTER(vp)],
            "ref_dense_features": [vp, f64, vp],
            "ref_dense_matvec": [vp, vp, vp],
        }.items():
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = args
        L.ref_free.argtypes = [vp]
        L.ref_forest_free.argtypes = [vp]
        L.ref_format.argtypes = [vp]
        L.ref_dims.argtypes = [vp, vp]
        L.ref_export.argtypes = [vp, vp, vp, vp]
        L.ref_forest_shape.argtypes = [vp, vp, vp, vp]
        L.ref_forest_export.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ref_predict_tree.argtypes = [vp, C.c_int, vp]
        L.ref_predict_forest.argtypes = [vp, vp]
        L.ref_format_feasible.argtypes = [C.c_int, vp, i64, f64, f64, i64]
        L.ref_rng_new.restype = vp
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_free.argtypes = [vp]
        L.ref_rng_next.restype = C.c_uint64
        L.ref_rng_next.argtypes = [vp]
        L.ref_rng_uniform_real.restype = f64
        L.ref_rng_uniform_real.argtypes = [vp, f64, f64]
        L.ref_rng_uniform_index.restype = C.c_uint64
        L.ref_rng_uniform_index.argtypes = [vp, C.c_uint64]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_random_vector.argtypes = [vp, i64, vp]
        _ref = L
    return _ref


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{status}] {msg}")
        self.status = status


def _rchk(st):
    if st != 0:
        raise RefError(st, ref().ref_last_error().decode())


# ======================================================= C restatement (oc_*)

class Rng:
    """mt19937_64 + rng.hpp draws, restated in C (oracle.c)."""

    def __init__(self, seed):
        self._buf = C.create_string_buffer(312 * 8 + 16)
        oc().oc_rng_seed(self._buf, C.c_uint64(seed))

    def next_u64(self):
        return oc().oc_rng_next(self._buf)

    def uniform_index(self, n):
        return oc().oc_rng_uniform_index(self._buf, n)

    def uniform_real(self, lo=0.0, hi=1.0):
        return oc().oc_rng_uniform_real(self._buf, lo, hi)

    def random_coo(self, max_dim=64, min_d=0.01, max_d=0.3):
        """tests/support/oracles.hpp:183-204 -> host COO dict (canonical)."""
        cap = max_dim * max_dim
        row = np.empty(cap, np.int64)
        col = np.empty(cap, np.int64)
        val = np.empty(cap, np.float64)
        n, m, z = i64(), i64(), i64()
        oc().oc_random_coo(self._buf, max_dim, min_d, max_d, C.byref(n), C.byref(m), C.byref(z),
                           _p(row), _p(col), _p(val))
        z = z.value
        return coo_dict(n.value, m.value, row[:z].copy(), col[:z].copy(), val[:z].copy())

    def random_vector(self, n):
        out = np.empty(n, np.float64)
        oc().oc_random_vector(self._buf, n, _p(out))
        return out


def derive_seed(seed, stream):
    return oc().oc_derive_seed(C.c_uint64(seed), C.c_uint64(stream))


def coo_dict(nrows, ncols, row, col, val):
    return {"format": COO, "nrows": int(nrows), "ncols": int(ncols),
            "row": np.asarray(row, np.int64), "col": np.asarray(col, np.int64),
            "val": np.asarray(val, np.float64)}


def from_triplets(nrows, ncols, row, col, val):
    """formats.cpp:293-322 (stable order for duplicate sums)."""
    row = np.array(row, np.int64)
    col = np.array(col, np.int64)
    val = np.array(val, np.float64)
    z = i64()
    st = oc().oc_from_triplets(nrows, ncols, row.size, _p(row), _p(col), _p(val), C.byref(z))
    if st != 0:
        raise RefError(st, "triplet outside matrix")
    z = z.value
    return coo_dict(nrows, ncols, row[:z], col[:z], val[:z])


def padded_entry_cap(cfg, nnz):
    return oc().oc_padded_entry_cap(cfg.get("max_padding_factor", 10.0),
                                    cfg.get("max_padded_entries", 0), nnz)


class PaddingOverflowOracle(Exception):
    pass


def oc_convert(coo, target, cfg=None):
    """from_coo (formats.cpp:411-430) on a canonical host COO dict."""
    cfg = cfg or {}
    L = oc()
    n, m = coo["nrows"], coo["ncols"]
    row, col, val = coo["row"], coo["col"], coo["val"]
    z = val.size
    if not L.oc_is_canonical(n, m, z, _p(row), _p(col)):
        raise RefError(1, "from_coo: source matrix is not canonical COO")
    cap = padded_entry_cap(cfg, z)
    base = {"format": target, "nrows": n, "ncols": m}
    if target == COO:
        return dict(coo)
    if target == CSR:
        rp = np.empty(n + 1, np.int64)
        L.oc_coo_to_csr(n, z, _p(row), _p(rp))
        base.update(row_ptr=rp, col=col.copy(), val=val.copy())
        return base
    if target == DIA:
        return dict(base, **_oc_dia(n, m, row, col, val, None, cap))
    if target == ELL:
        w = i64()
        if L.oc_ell_plan(n, z, _p(row), cap, C.byref(w)) == 2:
            raise PaddingOverflowOracle("ELL")
        w = w.value
        ec = np.empty(n * w, np.int64)
        ev = np.empty(n * w, np.float64)
        L.oc_ell_fill(n, z, _p(row), _p(col), _p(val), w, _p(ec), _p(ev))
        base.update(width=w, col=ec, val=ev, stored_nnz=z)
        return base
    if target == HYB:
        kh = L.oc_effective_kh(cfg.get("kh_override", 0), z, n)
        w, zc = i64(), i64()
        if L.oc_hyb_plan(n, z, _p(row), kh, cap, C.byref(w), C.byref(zc)) == 2:
            raise PaddingOverflowOracle("HYB")
        w, zc = w.value, zc.value
        ec = np.empty(n * w, np.int64)
        ev = np.empty(n * w, np.float64)
        cr, cc, cv = np.empty(zc, np.int64), np.empty(zc, np.int64), np.empty(zc, np.float64)
        L.oc_hyb_fill(n, z, _p(row), _p(col), _p(val), kh, w, _p(ec), _p(ev), _p(cr), _p(cc), _p(cv))
        base.update(kh=kh, ell={"width": w, "col": ec, "val": ev, "stored_nnz": z - zc},
                    coo={"row": cr, "col": cc, "val": cv})
        return base
    if target == HDC:
        thr = L.oc_true_diag_threshold(cfg.get("true_diag_ratio", 0.2), n, m)
        nd, zr = i64(), i64()
        offs = np.empty(max(n + m - 1, 1), np.int64)
        if L.oc_hdc_plan(n, m, z, _p(row), _p(col), thr, cap, C.byref(nd), _p(offs), C.byref(zr)) == 2:
            raise PaddingOverflowOracle("HDC")
        nd, zr = nd.value, zr.value
        offs = offs[:nd].copy()
        dv = np.empty(nd * n, np.float64)
        stored = i64()
        rp = np.empty(n + 1, np.int64)
        rc, rv = np.empty(zr, np.int64), np.empty(zr, np.float64)
        L.oc_hdc_fill(n, m, z, _p(row), _p(col), _p(val), thr, nd, _p(offs), _p(dv), C.byref(stored),
                      _p(rp), _p(rc), _p(rv))
        base.update(threshold=thr,
                    dia={"offsets": offs, "values": dv, "stored_nnz": stored.value},
                    csr={"row_ptr": rp, "col": rc, "val": rv})
        return base
    raise ValueError(target)


def _oc_dia(n, m, row, col, val, mask, cap):
    L = oc()
    z = val.size
    nd = i64()
    offs = np.empty(max(n + m - 1, 1), np.int64)
    if L.oc_dia_plan(n, m, z, _p(row), _p(col), _p(mask), cap, C.byref(nd), _p(offs)) == 2:
        raise PaddingOverflowOracle("DIA")
    nd = nd.value
    offs = offs[:nd].copy()
    vals = np.empty(nd * n, np.float64)
    stored = i64()
    L.oc_dia_fill(n, m, z, _p(row), _p(col), _p(val), _p(mask), nd, _p(offs), _p(vals), C.byref(stored))
    return {"offsets": offs, "values": vals, "stored_nnz": stored.value}


def oc_spmv(mat, x):
    """spmv (spmv.cpp:73-108, 191-208) on a host-layout dict."""
    L = oc()
    x = np.ascontiguousarray(x, np.float64)
    n, m = mat["nrows"], mat["ncols"]
    y = np.zeros(n, np.float64)
    f = mat["format"]

    def coo(d, acc):
        L.oc_spmv_coo(n, d["val"].size, _p(d["row"]), _p(d["col"]), _p(d["val"]), _p(x), _p(y), acc)

    def csr(d, acc):
        L.oc_spmv_csr(n, _p(d["row_ptr"]), _p(d["col"]), _p(d["val"]), _p(x), _p(y), acc)

    def dia(d, acc):
        L.oc_spmv_dia(n, m, d["offsets"].size, _p(d["offsets"]), _p(d["values"]), _p(x), _p(y), acc)

    def ell(d, acc):
        L.oc_spmv_ell(n, d["width"], _p(d["col"]), _p(d["val"]), _p(x), _p(y), acc)

    if f == COO:
        coo(mat, 0)
    elif f == CSR:
        csr(mat, 0)
    elif f == DIA:
        dia(mat, 0)
    elif f == ELL:
        ell(mat, 0)
    elif f == HYB:
        ell(mat["ell"], 0)
        coo(mat["coo"], 1)
    elif f == HDC:
        dia(mat["dia"], 0)
        csr(mat["csr"], 1)
    return y


class _View(C.Structure):
    _fields_ = [("format", C.c_int), ("nrows", i64), ("ncols", i64), ("coo_nnz", i64),
                ("coo_row", vp), ("coo_col", vp), ("csr_row_ptr", vp), ("csr_col", vp),
                ("ndiags", i64), ("offsets", vp), ("dia_values", vp), ("width", i64),
                ("ell_col", vp)]


def oc_features(mat, ratio=0.2):
    """extract_features (features.cpp:82-153) -> (row10 list, (visits, structure))."""
    v = _View()
    v.format = mat["format"]
    v.nrows, v.ncols = mat["nrows"], mat["ncols"]
    keep = []

    def set_coo(d):
        v.coo_nnz = d["val"].size
        v.coo_row, v.coo_col = _p(d["row"]), _p(d["col"])
        keep.append(d)

    def set_csr(d):
        v.csr_row_ptr, v.csr_col = _p(d["row_ptr"]), _p(d["col"])

    def set_dia(d):
        v.ndiags = d["offsets"].size
        v.offsets, v.dia_values = _p(d["offsets"]), _p(d["values"])

    def set_ell(d):
        v.width = d["width"]
        v.ell_col = _p(d["col"])

    f = mat["format"]
    {COO: lambda: set_coo(mat), CSR: lambda: set_csr(mat), DIA: lambda: set_dia(mat),
     ELL: lambda: set_ell(mat)}.get(f, lambda: None)()
    if f == HYB:
        set_ell(mat["ell"])
        set_coo(mat["coo"])
    if f == HDC:
        set_dia(mat["dia"])
        set_csr(mat["csr"])
    out = np.zeros(10, np.float64)
    stats = np.zeros(2, np.int64)
    st = oc().oc_extract_features(C.byref(v), ratio, _p(out), _p(stats))
    if st != 0:
        raise RefError(st, "extract_features")
    return out, (int(stats[0]), int(stats[1]))


def oc_predict_forest(ff, row10):
    """predict_forest (model.cpp:215-228); ff = FlatForest-like object."""
    row10 = np.ascontiguousarray(row10, np.float64)
    a = [np.ascontiguousarray(ff.node_off, np.int64), np.ascontiguousarray(ff.feature, np.int32),
         np.ascontiguousarray(ff.threshold, np.float64), np.ascontiguousarray(ff.left, np.int32),
         np.ascontiguousarray(ff.right, np.int32), np.ascontiguousarray(ff.cls, np.int32)]
    return oc().oc_predict_forest(ff.node_off.size - 1, *[_p(x) for x in a], _p(row10))


def oc_format_feasible(fmt, row10, cfg=None):
    cfg = cfg or {}
    row10 = np.ascontiguousarray(row10, np.float64)
    return bool(oc().oc_format_feasible(fmt, _p(row10), cfg.get("kh_override", 0),
                                        cfg.get("max_padding_factor", 10.0),
                                        cfg.get("max_padded_entries", 0)))


# ================================================= the reference (ref_*)

class RefMatrix:
    """A sparseoracle_ref::DynamicMatrix owned through the extern "C" shim."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            ref().ref_free(self.h)
        except Exception:
            pass

    @classmethod
    def from_triplets(cls, nrows, ncols, row, col, val):
        row, col, val = (np.ascontiguousarray(row, np.int64), np.ascontiguousarray(col, np.int64),
                         np.ascontiguousarray(val, np.float64))
        h = vp()
        _rchk(ref().ref_coo_from_triplets(nrows, ncols, val.size, _p(row), _p(col), _p(val), C.byref(h)))
        return cls(h)

    @classmethod
    def raw_coo(cls, nrows, ncols, row, col, val):
        row, col, val = (np.ascontiguousarray(row, np.int64), np.ascontiguousarray(col, np.int64),
                         np.ascontiguousarray(val, np.float64))
        h = vp()
        _rchk(ref().ref_coo_raw(nrows, ncols, val.size, _p(row), _p(col), _p(val), C.byref(h)))
        return cls(h)

    @classmethod
    def from_coo_dict(cls, d):
        return cls.raw_coo(d["nrows"], d["ncols"], d["row"], d["col"], d["val"])

    @staticmethod
    def _cfg(cfg):
        cfg = cfg or {}
        return (cfg.get("kh_override", 0), cfg.get("true_diag_ratio", 0.2),
                cfg.get("max_padding_factor", 10.0), cfg.get("max_padded_entries", 0))

    def from_coo(self, fmt, cfg=None):
        h = vp()
        _rchk(ref().ref_from_coo(self.h, fmt, *self._cfg(cfg), C.byref(h)))
        return RefMatrix(h)

    def switch_format(self, fmt, cfg=None):
        _rchk(ref().ref_switch_format(self.h, fmt, *self._cfg(cfg)))

    def to_coo(self):
        h = vp()
        _rchk(ref().ref_to_coo(self.h, C.byref(h)))
        return RefMatrix(h)

    def clone(self):
        h = vp()
        _rchk(ref().ref_clone(self.h, C.byref(h)))
        return RefMatrix(h)

    @property
    def format(self):
        return ref().ref_format(self.h)

    @property
    def dims(self):
        d = np.zeros(3, np.int64)
        ref().ref_dims(self.h, _p(d))
        return int(d[0]), int(d[1]), int(d[2])

    def export(self):
        """Copy of the active payload in the host-layout dict convention."""
        s = np.zeros(8, np.int64)
        arrs = (vp * 8)()
        lens = np.zeros(8, np.int64)
        ref().ref_export(self.h, _p(s), arrs, _p(lens))
        n, m, _ = self.dims

        def arr(i, dt):
            k = int(lens[i])
            if k == 0:
                return np.empty(0, dt)
            return np.ctypeslib.as_array(C.cast(arrs[i], C.POINTER(
                C.c_int64 if dt == np.int64 else C.c_double)), shape=(k,)).copy()

        f = self.format
        base = {"format": f, "nrows": n, "ncols": m}
        if f == COO:
            base.update(row=arr(0, np.int64), col=arr(1, np.int64), val=arr(2, np.float64))
        elif f == CSR:
            base.update(row_ptr=arr(0, np.int64), col=arr(1, np.int64), val=arr(2, np.float64))
        elif f == DIA:
            base.update(offsets=arr(0, np.int64), values=arr(1, np.float64), stored_nnz=int(s[0]))
        elif f == ELL:
            base.update(width=int(s[1]), col=arr(0, np.int64), val=arr(1, np.float64),
                        stored_nnz=int(s[0]))
        elif f == HYB:
            base.update(kh=int(s[2]),
                        ell={"width": int(s[1]), "col": arr(0, np.int64), "val": arr(1, np.float64),
                             "stored_nnz": int(s[0])},
                        coo={"row": arr(2, np.int64), "col": arr(3, np.int64), "val": arr(4, np.float64)})
        elif f == HDC:
            base.update(threshold=int(s[1]),
                        dia={"offsets": arr(0, np.int64), "values": arr(1, np.float64),
                             "stored_nnz": int(s[0])},
                        csr={"row_ptr": arr(2, np.int64), "col": arr(3, np.int64),
                             "val": arr(4, np.float64)})
        return base

    def spmv(self, x, nthreads=1):
        x = np.ascontiguousarray(x, np.float64)
        n, _, _ = self.dims
        y = np.empty(n, np.float64)
        _rchk(ref().ref_spmv(self.h, _p(x), x.size, _p(y), nthreads))
        return y

    def time_spmv(self, x, reps, nthreads=1):
        x = np.ascontiguousarray(x, np.float64)
        per = np.empty(reps, np.float64)
        tot = np.zeros(1, np.float64)
        _rchk(ref().ref_time_spmv(self.h, _p(x), x.size, reps, nthreads, _p(per), _p(tot)))
        return per, float(tot[0])

    def extract_features(self, ratio=0.2):
        out = np.zeros(10, np.float64)
        st = np.zeros(2, np.int64)
        _rchk(ref().ref_extract_features(self.h, ratio, _p(out), _p(st)))
        return out, (int(st[0]), int(st[1]))

    def dense_features(self, ratio=0.2):
        out = np.zeros(10, np.float64)
        _rchk(ref().ref_dense_features(self.h, ratio, _p(out)))
        return out

    def dense_matvec(self, x):
        x = np.ascontiguousarray(x, np.float64)
        n, _, _ = self.dims
        y = np.empty(n, np.float64)
        _rchk(ref().ref_dense_matvec(self.h, _p(x), _p(y)))
        return y


class RefRng:
    """The reference's own Rng (rng.hpp) through the shim."""

    def __init__(self, seed):
        self.h = ref().ref_rng_new(C.c_uint64(seed))

    def __del__(self):
        try:
            ref().ref_rng_free(self.h)
        except Exception:
            pass

    def next_u64(self):
        return ref().ref_rng_next(self.h)

    def uniform_real(self, lo=0.0, hi=1.0):
        return ref().ref_rng_uniform_real(self.h, lo, hi)

    def uniform_index(self, n):
        return ref().ref_rng_uniform_index(self.h, n)

    def random_coo(self, max_dim=64, min_d=0.01, max_d=0.3):
        h = vp()
        _rchk(ref().ref_random_coo(self.h, max_dim, min_d, max_d, C.byref(h)))
        return RefMatrix(h)

    def random_vector(self, n):
        out = np.empty(n, np.float64)
        ref().ref_random_vector(self.h, n, _p(out))
        return out


def ref_band_matrix(n, half_band):
    h = vp()
    _rchk(ref().ref_band_matrix(n, half_band, C.byref(h)))
    return RefMatrix(h)


class RefForest:
    def __init__(self, ff):
        a = [np.ascontiguousarray(ff.node_off, np.int64), np.ascontiguousarray(ff.feature, np.int32),
             np.ascontiguousarray(ff.threshold, np.float64), np.ascontiguousarray(ff.left, np.int32),
             np.ascontiguousarray(ff.right, np.int32), np.ascontiguousarray(ff.cls, np.int32)]
        counts = ff.counts if ff.counts is not None else np.ones((a[1].size, 6), np.int64)
        counts = np.ascontiguousarray(counts, np.int64)
        h = vp()
        _rchk(ref().ref_forest_create(ff.kind, a[0].size - 1, *[_p(x) for x in a], _p(counts), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            ref().ref_forest_free(self.h)
        except Exception:
            pass

    def predict_forest(self, row10):
        return ref().ref_predict_forest(self.h, _p(np.ascontiguousarray(row10, np.float64)))

    def predict_tree(self, t, row10):
        return ref().ref_predict_tree(self.h, t, _p(np.ascontiguousarray(row10, np.float64)))


def ref_tune_ml(m: RefMatrix, forest: RefForest, ratio=0.2, cfg=None):
    cfg = cfg or {}
    out = np.zeros(4, np.int32)
    t = np.zeros(2, np.float64)
    _rchk(ref().ref_tune_ml(m.h, forest.h, ratio, cfg.get("kh_override", 0),
                            cfg.get("max_padding_factor", 10.0), cfg.get("max_padded_entries", 0),
                            _p(out), _p(t)))
    return {"chosen": int(out[0]), "source": int(out[1]), "switched": bool(out[2]),
            "fallback_csr": bool(out[3]), "t_fe": float(t[0]), "t_pred": float(t[1])}
