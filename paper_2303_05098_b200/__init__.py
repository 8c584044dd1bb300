"""B200-native (sm_100a) Morpheus-Oracle hot path.

Device-resident sparse containers in six formats, CSR->format conversion
kernels, fused feature extraction, on-device tree/forest prediction and fp64
SpMV, behind the reference's C++ API (include/sparseoracle/*.hpp, implemented
in cpp/ over the C-ABI include/sparseoracle_b200.h).  This Python package is
the ctypes view of the same C-ABI used by the tests and bench.py.
"""
from .device import (COO, CSR, DIA, ELL, FORMAT_NAMES, HDC, HYB, AllFormatsInfeasible,
                     ConversionConfig, DeviceForest, DeviceMatrix, DimensionMismatch,
                     EmptyMatrix, Error, FeatureVector, FlatForest, IndexOutOfRange,
                     InvalidInput, MalformedModel, OutOfMemory, PaddingOverflow, ParseError,
                     UnsupportedFormat, collapse_label, format_feasible, kernel_twins, set_device,
                     tune_ml)

__all__ = ["COO", "CSR", "DIA", "ELL", "HYB", "HDC", "FORMAT_NAMES", "DeviceMatrix",
           "DeviceForest", "FlatForest", "ConversionConfig", "FeatureVector", "tune_ml",
           "format_feasible", "set_device", "Error", "InvalidInput", "PaddingOverflow",
           "DimensionMismatch", "EmptyMatrix", "MalformedModel", "IndexOutOfRange",
           "AllFormatsInfeasible", "ParseError", "UnsupportedFormat", "OutOfMemory", "kernel_twins",
           "collapse_label"]
