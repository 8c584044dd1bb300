"""ctypes binding of the C-ABI in include/sparseoracle_b200.h.

The shared library is built in-tree (``make`` at the repo root) into
``paper_2303_05098_b200/lib/libsparseoracle_b200.so``.  There is no CPU
fallback: if the library cannot be loaded, importing the matrix API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, "lib", "libsparseoracle_b200.so")
CPP_LIB_PATH = os.path.join(_HERE, "lib", "libsparseoracle.so")

_lock = threading.Lock()
_lib = None

i64 = C.c_int64
i32 = C.c_int32
f64 = C.c_double
P = C.POINTER
vp = C.c_void_p


class ConversionConfig(C.Structure):
    """formats.hpp:124-139 ConversionConfig."""

    _fields_ = [("kh_override", i64), ("true_diag_ratio", f64),
                ("max_padding_factor", f64), ("max_padded_entries", i64)]

    def __init__(self, kh_override=0, true_diag_ratio=0.2, max_padding_factor=10.0,
                 max_padded_entries=0):
        super().__init__(kh_override, true_diag_ratio, max_padding_factor, max_padded_entries)


class FeatureVector(C.Structure):
    """features.hpp:12-23, fields in struct order."""

    _fields_ = [("nrows", i64), ("ncols", i64), ("nnz", i64), ("avg_nnz_per_row", f64),
                ("density", f64), ("max_nnz_per_row", i64), ("min_nnz_per_row", i64),
                ("nnz_row_spread", f64), ("ndiags", i64), ("ntrue_diags", i64)]

    def to_row(self):
        """features_to_row order (features.cpp:155-166)."""
        return [float(self.nrows), float(self.ncols), float(self.nnz), self.avg_nnz_per_row,
                self.density, float(self.max_nnz_per_row), float(self.min_nnz_per_row),
                self.nnz_row_spread, float(self.ndiags), float(self.ntrue_diags)]

    @classmethod
    def from_row(cls, row):
        """row_to_features (features.cpp:168-181)."""
        r = [float(v) for v in row]
        return cls(int(r[0]), int(r[1]), int(r[2]), r[3], r[4], int(r[5]), int(r[6]), r[7],
                   int(r[8]), int(r[9]))


class ScanStats(C.Structure):
    _fields_ = [("entry_visits", i64), ("structure_reads", i64)]


class MatrixInfo(C.Structure):
    _fields_ = [("format", i32), ("device", i32), ("nrows", i64), ("ncols", i64), ("nnz", i64),
                ("coo_nnz", i64), ("csr_nnz", i64), ("ndiags", i64), ("dia_stored_nnz", i64),
                ("ell_width", i64), ("ell_stored_nnz", i64), ("kh", i64),
                ("true_diag_threshold", i64)]


class HostArrays(C.Structure):
    _fields_ = [("coo_row", vp), ("coo_col", vp), ("coo_val", vp), ("csr_row_ptr", vp),
                ("csr_col", vp), ("csr_val", vp), ("dia_offsets", vp), ("dia_values", vp),
                ("ell_col", vp), ("ell_val", vp)]


class TuneOutcome(C.Structure):
    _fields_ = [("chosen", i32), ("source", i32), ("switched", i32), ("fallback_csr", i32),
                ("feature_time_seconds", f64), ("predict_time_seconds", f64),
                ("features", FeatureVector), ("wall_time_seconds", f64)]


# function name -> (restype, argtypes)
_SIGS = {
    "so_last_error": (C.c_char_p, []),
    "so_version": (C.c_char_p, []),
    "so_kernel_launches": (C.c_int64, []),
    "so_get_device": (C.c_int, [P(C.c_int)]),
    "so_set_device": (C.c_int, [C.c_int]),
    "so_device_sync": (C.c_int, []),
    "so_default_stream": (vp, []),
    "so_matrix_upload_coo": (C.c_int, [i64, i64, i64, vp, vp, vp, P(vp)]),
    "so_matrix_upload_csr": (C.c_int, [i64, i64, i64, vp, vp, vp, P(vp)]),
    "so_matrix_upload_dia": (C.c_int, [i64, i64, i64, vp, vp, i64, P(vp)]),
    "so_matrix_upload_ell": (C.c_int, [i64, i64, i64, vp, vp, i64, P(vp)]),
    "so_matrix_upload_hyb": (C.c_int, [i64, i64, i64, vp, vp, i64, i64, vp, vp, vp, i64, P(vp)]),
    "so_matrix_upload_hdc": (C.c_int, [i64, i64, i64, vp, vp, i64, i64, vp, vp, vp, i64, P(vp)]),
    "so_coo_from_triplets": (C.c_int, [i64, i64, i64, vp, vp, vp, P(vp)]),
    "so_read_matrix_market": (C.c_int, [C.c_char_p, P(vp)]),
    "so_write_matrix_market": (C.c_int, [vp, C.c_char_p]),
    "so_matrix_import_csr_device": (C.c_int, [i64, i64, i64, vp, vp, vp, P(vp)]),
    "so_matrix_free": (None, [vp]),
    "so_matrix_info_get": (C.c_int, [vp, P(MatrixInfo)]),
    "so_matrix_download": (C.c_int, [vp, P(HostArrays)]),
    "so_from_coo": (C.c_int, [vp, i32, P(ConversionConfig), P(vp)]),
    "so_convert": (C.c_int, [vp, i32, P(ConversionConfig), P(vp)]),
    "so_to_coo": (C.c_int, [vp, P(vp)]),
    "so_format_feasible": (i32, [i32, P(FeatureVector), P(ConversionConfig)]),
    "so_spmv_device": (C.c_int, [vp, vp, vp, vp]),
    "so_spmv_device_rows": (C.c_int, [vp, vp, vp, i64, i64, vp]),
    "so_spmv_rows_push": (C.c_int, [vp, vp, vp, i64, i64, vp, vp, vp, C.c_uint64, vp]),
    "so_wait_flag": (C.c_int, [vp, C.c_uint64, vp]),
    "so_wait_flag_timeouts": (C.c_int64, []),
    "so_ipc_alloc": (C.c_int, [i64, C.POINTER(vp), C.c_char_p]),
    "so_ipc_open": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "so_ipc_close": (C.c_int, [vp]),
    "so_ipc_free": (C.c_int, [vp]),
    "so_gen_stencil27_dia": (C.c_int, [i64, i64, i64, i64, i64, C.c_uint64, P(vp)]),
    "so_spmv": (C.c_int, [vp, vp, i64, vp]),
    "so_spmv_new": (C.c_int, [vp, vp, i64, vp, vp]),
    "so_time_spmv": (C.c_int, [vp, vp, i64, i64, vp, P(f64)]),
    "so_spmv_bytes": (i64, [vp]),
    "so_extract_features": (C.c_int, [vp, f64, P(FeatureVector), P(ScanStats)]),
    "so_forest_upload": (C.c_int, [i32, i32, vp, vp, vp, vp, vp, vp, P(vp)]),
    "so_forest_free": (None, [vp]),
    "so_predict": (C.c_int, [vp, P(FeatureVector), P(i32)]),
    "so_predict_rows": (C.c_int, [vp, i64, vp, vp]),
    "so_predict_rows_latency": (C.c_int, [vp, i64, vp, vp]),
    "so_tune_ml": (C.c_int, [vp, vp, f64, P(ConversionConfig), P(TuneOutcome)]),
    "so_dist_create": (C.c_int, [vp, i32, i32, i32, vp, i64, P(vp)]),
    "so_dist_handle": (C.c_int, [vp, C.c_char_p]),
    "so_dist_connect": (C.c_int, [vp, C.c_char_p]),
    "so_dist_x": (C.c_int, [vp, i32, P(vp), P(i64), P(i64)]),
    "so_dist_iterate": (C.c_int, [vp, i64, vp]),
    "so_dist_timeouts": (C.c_int64, []),
    "so_dist_free": (None, [vp]),
}


# so_make_output: double* (*)(void* ctx, int64_t nrows)
MAKE_OUTPUT = C.CFUNCTYPE(vp, vp, i64)


def exported_symbols():
    return sorted(_SIGS)


def build():
    """Compile the CUDA library in-tree (nvcc, sm_100a)."""
    subprocess.run(["make", "-C", _REPO, "-j8"], check=True, stdout=subprocess.DEVNULL)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            h = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
        return _lib
