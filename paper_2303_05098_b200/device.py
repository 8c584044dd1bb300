"""Python handle layer over the C-ABI (tests, bench, tools).

Mirrors the reference's operator surface for this path -- containers,
``from_coo`` / ``switch_format`` / ``to_coo``, ``spmv`` / ``time_spmv``,
``extract_features``, ``predict_forest``, ``tune_ml``, ``format_feasible`` --
with the same argument meaning and the same error types
(proj/include/sparseoracle/*.hpp).  Every call goes to the sm_100a library;
there is no host compute path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi as A

COO, CSR, DIA, ELL, HYB, HDC = range(6)
FORMAT_NAMES = ("COO", "CSR", "DIA", "ELL", "HYB", "HDC")


# ---------------------------------------------------------------- errors
# errors.hpp:8-71
class Error(RuntimeError):
    pass


class InvalidInput(Error):
    pass


class PaddingOverflow(Error):
    pass


class DimensionMismatch(Error):
    pass


class EmptyMatrix(Error):
    pass


class MalformedModel(Error):
    pass


class IndexOutOfRange(Error):
    pass


class AllFormatsInfeasible(Error):
    pass


class CudaError(Error):
    pass


class ParseError(Error):
    pass


class UnsupportedFormat(Error):
    pass


class OutOfMemory(Error):
    pass


_STATUS = {1: InvalidInput, 2: PaddingOverflow, 3: DimensionMismatch, 4: EmptyMatrix,
           5: MalformedModel, 6: IndexOutOfRange, 7: AllFormatsInfeasible, 8: CudaError,
           9: OutOfMemory, 10: Error, 11: ParseError, 12: UnsupportedFormat}


def _check(st):
    if st != 0:
        msg = A.lib().so_last_error().decode(errors="replace")
        raise _STATUS.get(st, Error)(msg)


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


ConversionConfig = A.ConversionConfig
FeatureVector = A.FeatureVector


# ---------------------------------------------------------------- matrices
class DeviceMatrix:
    """A device-resident matrix in one of the six formats (DynamicMatrix payload)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self._keep = None

    def __del__(self):
        try:
            if self._h:
                A.lib().so_matrix_free(self._h)
                self._h = C.c_void_p(0)
        except Exception:
            pass

    # -- construction (host arrays in the reference layout) ----------------
    @classmethod
    def coo(cls, nrows, ncols, row, col, val):
        row, col, val = _i64(row), _i64(col), _f64(val)
        out = C.c_void_p()
        _check(A.lib().so_matrix_upload_coo(nrows, ncols, val.size, _ptr(row), _ptr(col), _ptr(val),
                                            C.byref(out)))
        return cls(out)

    @classmethod
    def from_triplets(cls, nrows, ncols, row, col, val):
        """CooMatrix::from_triplets on the device -> canonical COO."""
        row, col, val = _i64(row), _i64(col), _f64(val)
        out = C.c_void_p()
        _check(A.lib().so_coo_from_triplets(nrows, ncols, val.size, _ptr(row), _ptr(col), _ptr(val),
                                            C.byref(out)))
        return cls(out)

    @classmethod
    def read_matrix_market(cls, path):
        """read_matrix_market (ingest.cpp:135-208): host-parallel parse, device
        canonicalization -> canonical COO.  Raises ParseError /
        UnsupportedFormat / IndexOutOfRange like the reference."""
        out = C.c_void_p()
        _check(A.lib().so_read_matrix_market(str(path).encode(), C.byref(out)))
        return cls(out)

    def write_matrix_market(self, path):
        """write_matrix_market (ingest.cpp:210-224) of a canonical COO."""
        _check(A.lib().so_write_matrix_market(self._h, str(path).encode()))

    @classmethod
    def csr(cls, nrows, ncols, row_ptr, col, val):
        row_ptr, col, val = _i64(row_ptr), _i64(col), _f64(val)
        out = C.c_void_p()
        _check(A.lib().so_matrix_upload_csr(nrows, ncols, val.size, _ptr(row_ptr), _ptr(col),
                                            _ptr(val), C.byref(out)))
        return cls(out)

    @classmethod
    def csr_device(cls, nrows, ncols, nnz, row_ptr_ptr, col_ptr, val_ptr):
        """Import a CSR that already lives in device memory (int64 row_ptr,
        int32 col, f64 val device pointers, e.g. torch tensors' data_ptr())."""
        out = C.c_void_p()
        _check(A.lib().so_matrix_import_csr_device(nrows, ncols, nnz, C.c_void_p(row_ptr_ptr),
                                                   C.c_void_p(col_ptr), C.c_void_p(val_ptr), C.byref(out)))
        return cls(out)

    @classmethod
    def dia(cls, nrows, ncols, offsets, values, stored_nnz):
        offsets, values = _i64(offsets), _f64(values)
        out = C.c_void_p()
        _check(A.lib().so_matrix_upload_dia(nrows, ncols, offsets.size, _ptr(offsets), _ptr(values),
                                            int(stored_nnz), C.byref(out)))
        return cls(out)

    @classmethod
    def ell(cls, nrows, ncols, width, col, val, stored_nnz):
        col, val = _i64(col), _f64(val)
        out = C.c_void_p()
        _check(A.lib().so_matrix_upload_ell(nrows, ncols, width, _ptr(col), _ptr(val),
                                            int(stored_nnz), C.byref(out)))
        return cls(out)

    @classmethod
    def from_host(cls, m: dict):
        """Upload a reference-layout dict (see ``download``)."""
        f = m["format"]
        n, nc = m["nrows"], m["ncols"]
        if f == COO:
            return cls.coo(n, nc, m["row"], m["col"], m["val"])
        if f == CSR:
            return cls.csr(n, nc, m["row_ptr"], m["col"], m["val"])
        if f == DIA:
            return cls.dia(n, nc, m["offsets"], m["values"], m["stored_nnz"])
        if f == ELL:
            return cls.ell(n, nc, m["width"], m["col"], m["val"], m["stored_nnz"])
        out = C.c_void_p()
        if f == HYB:
            e, c = m["ell"], m["coo"]
            ec, ev = _i64(e["col"]), _f64(e["val"])
            cr, cc, cv = _i64(c["row"]), _i64(c["col"]), _f64(c["val"])
            _check(A.lib().so_matrix_upload_hyb(n, nc, e["width"], _ptr(ec), _ptr(ev),
                                                int(e["stored_nnz"]), cv.size, _ptr(cr), _ptr(cc),
                                                _ptr(cv), int(m["kh"]), C.byref(out)))
            return cls(out)
        if f == HDC:
            d, c = m["dia"], m["csr"]
            do, dv = _i64(d["offsets"]), _f64(d["values"])
            rp, cc, cv = _i64(c["row_ptr"]), _i64(c["col"]), _f64(c["val"])
            _check(A.lib().so_matrix_upload_hdc(n, nc, do.size, _ptr(do), _ptr(dv),
                                                int(d["stored_nnz"]), cv.size, _ptr(rp), _ptr(cc),
                                                _ptr(cv), int(m["threshold"]), C.byref(out)))
            return cls(out)
        raise InvalidInput(f"unknown format {f}")

    # -- introspection -------------------------------------------------------
    @property
    def info(self) -> A.MatrixInfo:
        i = A.MatrixInfo()
        _check(A.lib().so_matrix_info_get(self._h, C.byref(i)))
        return i

    @property
    def format(self):
        return self.info.format

    @property
    def nrows(self):
        return self.info.nrows

    @property
    def ncols(self):
        return self.info.ncols

    def nnz(self):
        return self.info.nnz

    def download(self) -> dict:
        """Host arrays in the reference layout (int64 indices, row-major ELL)."""
        i = self.info
        n = i.nrows
        h = A.HostArrays()
        a = {}

        def alloc(name, count, dt):
            arr = np.empty(int(count), dtype=dt)
            a[name] = arr
            setattr(h, name, arr.ctypes.data if arr.size else None)
            return arr

        f = i.format
        if f in (COO, HYB):
            alloc("coo_row", i.coo_nnz, np.int64)
            alloc("coo_col", i.coo_nnz, np.int64)
            alloc("coo_val", i.coo_nnz, np.float64)
        if f in (CSR, HDC):
            alloc("csr_row_ptr", n + 1, np.int64)
            alloc("csr_col", i.csr_nnz, np.int64)
            alloc("csr_val", i.csr_nnz, np.float64)
        if f in (DIA, HDC):
            alloc("dia_offsets", i.ndiags, np.int64)
            alloc("dia_values", i.ndiags * n, np.float64)
        if f in (ELL, HYB):
            alloc("ell_col", i.ell_width * n, np.int64)
            alloc("ell_val", i.ell_width * n, np.float64)
        _check(A.lib().so_matrix_download(self._h, C.byref(h)))
        base = {"format": f, "nrows": n, "ncols": i.ncols}
        coo = lambda: {"row": a["coo_row"], "col": a["coo_col"], "val": a["coo_val"]}
        csr = lambda: {"row_ptr": a["csr_row_ptr"], "col": a["csr_col"], "val": a["csr_val"]}
        dia = lambda: {"offsets": a["dia_offsets"], "values": a["dia_values"],
                       "stored_nnz": i.dia_stored_nnz}
        ell = lambda: {"width": i.ell_width, "col": a["ell_col"], "val": a["ell_val"],
                       "stored_nnz": i.ell_stored_nnz}
        if f == COO:
            base.update(coo())
        elif f == CSR:
            base.update(csr())
        elif f == DIA:
            base.update(dia())
        elif f == ELL:
            base.update(ell())
        elif f == HYB:
            base.update({"ell": ell(), "coo": coo(), "kh": i.kh})
        elif f == HDC:
            base.update({"dia": dia(), "csr": csr(), "threshold": i.true_diag_threshold})
        return base

    # -- conversions (formats.cpp:411-467) ---------------------------------
    def from_coo(self, target, config: ConversionConfig | None = None):
        cfg = config or ConversionConfig()
        out = C.c_void_p()
        _check(A.lib().so_from_coo(self._h, int(target), C.byref(cfg), C.byref(out)))
        return DeviceMatrix(out)

    def convert(self, target, config: ConversionConfig | None = None):
        cfg = config or ConversionConfig()
        out = C.c_void_p()
        _check(A.lib().so_convert(self._h, int(target), C.byref(cfg), C.byref(out)))
        return DeviceMatrix(out)

    def to_coo(self):
        out = C.c_void_p()
        _check(A.lib().so_to_coo(self._h, C.byref(out)))
        return DeviceMatrix(out)

    # -- SpMV (spmv.hpp:20-32) --------------------------------------------
    def spmv(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(max(self.nrows, 0), dtype=np.float64)
        _check(A.lib().so_spmv(self._h, _ptr(x), x.size, _ptr(y)))
        return y

    def spmv_new(self, x, fail_alloc=False) -> np.ndarray:
        """so_spmv_new: y's storage comes from a callback the library calls
        on this thread while the device works (the C++ spmv(m, x) path)."""
        x = _f64(x)
        out = {}

        def make(_ctx, n):
            if fail_alloc:
                return None
            out["y"] = np.zeros(n, dtype=np.float64)  # value-initialised, like std::vector
            return out["y"].ctypes.data

        cb = A.MAKE_OUTPUT(make)
        _check(A.lib().so_spmv_new(self._h, _ptr(x), x.size, C.cast(cb, C.c_void_p), None))
        return out["y"]

    def spmv_into(self, x_host: np.ndarray, y_host: np.ndarray):
        """spmv with caller-owned (ideally pinned) host buffers."""
        _check(A.lib().so_spmv(self._h, C.c_void_p(x_host.ctypes.data), x_host.size,
                               C.c_void_p(y_host.ctypes.data)))

    @classmethod
    def stencil27(cls, g, row_lo=0, row_hi=None, col_lo=0, col_hi=None, seed=5):
        """Device-generated 27-point stencil slice (DIA), see so_gen_stencil27_dia."""
        n = g ** 3
        out = C.c_void_p()
        _check(A.lib().so_gen_stencil27_dia(g, row_lo, n if row_hi is None else row_hi, col_lo,
                                            n if col_hi is None else col_hi, seed, C.byref(out)))
        return cls(out)

    def spmv_device_rows(self, x_ptr: int, y_ptr: int, row_lo: int, row_hi: int, stream: int | None = None):
        _check(A.lib().so_spmv_device_rows(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), int(row_lo),
                                           int(row_hi), C.c_void_p(stream or 0)))

    def spmv_device(self, x_ptr: int, y_ptr: int, stream: int | None = None):
        _check(A.lib().so_spmv_device(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                      C.c_void_p(stream or 0)))

    def time_spmv(self, x, reps):
        x = _f64(x)
        per = np.zeros(max(int(reps), 1), dtype=np.float64)
        tot = C.c_double()
        _check(A.lib().so_time_spmv(self._h, _ptr(x), x.size, int(reps), _ptr(per), C.byref(tot)))
        return per, tot.value

    @property
    def spmv_bytes(self) -> int:
        return int(A.lib().so_spmv_bytes(self._h))

    # -- features (features.hpp:33-42) ---------------------------------------
    def extract_features(self, true_diag_ratio=0.2, with_stats=False):
        f = A.FeatureVector()
        st = A.ScanStats()
        _check(A.lib().so_extract_features(self._h, float(true_diag_ratio), C.byref(f), C.byref(st)))
        return (f, st) if with_stats else f


# ---------------------------------------------------------------- forests
@dataclass
class FlatForest:
    """Flat SoA forest; tree t owns nodes [node_off[t], node_off[t+1])."""

    kind: int  # 0 tree, 1 forest (model.hpp:37)
    node_off: np.ndarray
    feature: np.ndarray
    threshold: np.ndarray
    left: np.ndarray
    right: np.ndarray
    cls: np.ndarray
    counts: np.ndarray | None = None

    @property
    def n_trees(self):
        return int(self.node_off.size - 1)


class DeviceForest:
    def __init__(self, ff: FlatForest):
        self.flat = ff
        out = C.c_void_p()
        arrs = [np.ascontiguousarray(ff.node_off, np.int64),
                np.ascontiguousarray(ff.feature, np.int32),
                np.ascontiguousarray(ff.threshold, np.float64),
                np.ascontiguousarray(ff.left, np.int32),
                np.ascontiguousarray(ff.right, np.int32),
                np.ascontiguousarray(ff.cls, np.int32)]
        _check(A.lib().so_forest_upload(ff.kind, ff.n_trees, *[_ptr(a) for a in arrs], C.byref(out)))
        self._h = out

    def __del__(self):
        try:
            if self._h:
                A.lib().so_forest_free(self._h)
        except Exception:
            pass

    def predict(self, fv: FeatureVector) -> int:
        """predict_forest (model.cpp:215-228): plurality over all trees, ties -> lowest id."""
        out = C.c_int32()
        _check(A.lib().so_predict(self._h, C.byref(fv), C.byref(out)))
        return out.value

    def predict_rows(self, rows) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 10)
        out = np.empty(rows.shape[0], dtype=np.int32)
        _check(A.lib().so_predict_rows(self._h, rows.shape[0], _ptr(rows), _ptr(out)))
        return out

    def predict_rows_latency(self, rows) -> np.ndarray:
        """The fused tuner's single-row path (blocked warp walk), one CTA per row."""
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 10)
        out = np.empty(rows.shape[0], dtype=np.int32)
        _check(A.lib().so_predict_rows_latency(self._h, rows.shape[0], _ptr(rows), _ptr(out)))
        return out


def kernel_twins(mats: dict) -> dict:
    """Formats whose multiply runs the very same kernel on the very same
    arrays as another format of the same matrix ({format: twin}): HDC with
    an empty CSR part and every diagonal kept is the DIA kernel on the DIA
    arrays, HDC with no diagonal at all is the CSR kernel on the CSR arrays,
    HYB with an empty COO part and the ELL width is the ELL kernel on the ELL
    arrays (spmv.cu spmv_device).  `mats` maps format id -> DeviceMatrix of
    one matrix (infeasible formats absent).  A measured "optimum" between
    twins is timing noise, so labels and accuracy treat them as one class."""
    tw = {}
    if DIA in mats and HDC in mats:
        a, b = mats[DIA].info, mats[HDC].info
        if b.csr_nnz == 0 and b.ndiags == a.ndiags:
            tw[HDC], tw[DIA] = DIA, HDC
    if CSR in mats and HDC in mats and HDC not in tw:
        if mats[HDC].info.ndiags == 0:
            tw[HDC], tw[CSR] = CSR, HDC
    if ELL in mats and HYB in mats:
        a, b = mats[ELL].info, mats[HYB].info
        if b.coo_nnz == 0 and b.ell_width == a.ell_width:
            tw[HYB], tw[ELL] = ELL, HYB
    return tw


def collapse_label(label: int, twins: dict) -> int:
    """The lowest id of a format's twin class (the reference's argmin breaks
    exact ties toward the lowest FormatId, pipeline.cpp:95-104)."""
    return min(label, twins.get(label, label))


def tune_ml(m: DeviceMatrix, forest: DeviceForest, true_diag_ratio=0.2,
            config: ConversionConfig | None = None) -> A.TuneOutcome:
    """tune_ml (tuners.cpp:92-114) fully on the device."""
    cfg = config or ConversionConfig()
    o = A.TuneOutcome()
    _check(A.lib().so_tune_ml(m._h, forest._h, float(true_diag_ratio), C.byref(cfg), C.byref(o)))
    return o


def format_feasible(target, f: FeatureVector, config: ConversionConfig | None = None) -> bool:
    cfg = config or ConversionConfig()
    return bool(A.lib().so_format_feasible(int(target), C.byref(f), C.byref(cfg)))


def set_device(d: int):
    _check(A.lib().so_set_device(int(d)))
