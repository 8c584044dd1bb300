"""The reference's CSV wire formats for profiling and feature data
(ingest.cpp:419-470, pipeline.cpp:71-130), written from B200 measurements so
the reference's own tooling -- read_profile_csv, read_feature_csv,
build_training_csv and cmd_train (pipeline.cpp:190-252) -- consumes B200
labels unchanged.  Host-side text, no compute.

  profile CSV:  matrix_id,format_id,repetitions,total_seconds,feasible
  feature CSV:  matrix_id,M,N,NNZ,avg_nnz,density,max_nnz,min_nnz,
                nnz_spread,ndiags,ntrue_diags
Doubles use the shortest round-trip text of std::to_chars (format_double,
model.cpp:195-200); counts are written as integers.
"""
from __future__ import annotations

from .forest import format_double

PROFILE_HEADER = "matrix_id,format_id,repetitions,total_seconds,feasible"
FEATURE_HEADER = ("matrix_id,M,N,NNZ,avg_nnz,density,max_nnz,min_nnz,nnz_spread,ndiags,"
                  "ntrue_diags")
_INT_FIELDS = (0, 1, 2, 5, 6, 8, 9)  # features_to_row positions written as index_t


def write_profile_csv(path, records):
    """records: iterable of (matrix_id, format_id, repetitions, total_seconds,
    feasible); an infeasible format (PaddingOverflow) has total 0 and feasible
    0, as cmd_profile writes it (pipeline.cpp:84-95)."""
    lines = [PROFILE_HEADER]
    for mid, fmt, reps, total, feas in records:
        if "," in str(mid):
            raise ValueError("matrix_id must not contain ','")
        lines.append(f"{mid},{int(fmt)},{int(reps)},{format_double(float(total) if feas else 0.0)},"
                     f"{1 if feas else 0}")
    with open(path, "w", newline="\n") as f:
        f.write("\n".join(lines) + "\n")


def write_feature_csv(path, rows):
    """rows: iterable of (matrix_id, row10) with row10 = features_to_row
    (FeatureVector.to_row())."""
    lines = [FEATURE_HEADER]
    for mid, r in rows:
        if len(r) != 10:
            raise ValueError("feature rows have 10 fields")
        fields = [str(int(r[k])) if k in _INT_FIELDS else format_double(float(r[k])) for k in range(10)]
        lines.append(f"{mid}," + ",".join(fields))
    with open(path, "w", newline="\n") as f:
        f.write("\n".join(lines) + "\n")
