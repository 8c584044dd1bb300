#!/usr/bin/env python3
"""The reference CPU path per format and config:
the reference's own sources compiled in place (oracle/_ref, -O3 -DNDEBUG, no
-march, as its Release build), timed on THIS host with its own entry points:

* from_coo conversion per format (formats.cpp:411-430), PaddingOverflow =
  infeasible;
* time_spmv(m, x = ones, reps, nthreads) (spmv.cpp:221-246) at nthreads = 1
  and nthreads = hardware threads, reps so each total is >= ~1 s (bounded);
* extract_features (features.cpp:82-153) and predict_forest
  (model.cpp:215-228, the shipped forest) with steady_clock / perf_counter;
* the tuning cost in CSR-SpMV equivalents (pipeline.cpp:300-302) and the
  Eq. 2 speedup at 1000 repetitions (pipeline.cpp:298-299), single thread as
  the reference tuner runs (TunerConfig nthreads = 1).

GB/s use the algorithmic bytes of DESIGN.md §4 (computed here from the
reference's own converted arrays, pure numpy), GFLOP/s = 2 z / t.
Configs 1-3 at full size, config 5 at 128^3 (512^3 does not materialise
through the CPU path; stated).  Measurement script (test infrastructure may
be imported here: it times the reference, it is not the product path).

    python scripts/cpu_baseline.py [--configs 1,2,3,5] [--budget 1.0] > profiles/rNN_cpu_baseline.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import oracle as O  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402

FMT = ("COO", "CSR", "DIA", "ELL", "HYB", "HDC")


def algorithmic_bytes(e):
    """DESIGN.md §4 / so_spmv_bytes from the reference's exported arrays."""
    n, m = e["nrows"], e["ncols"]
    xy = 8 * m + 8 * n

    def dia(d):
        offs = d["offsets"]
        cells = sum(max(0, min(n, m - int(o)) - max(0, -int(o))) for o in offs)
        return 8 * cells + 8 * offs.size

    def ell(d):
        w = d["width"]
        if w == 0:
            return 0
        col = d["col"].reshape(n, w)
        live = col != -1
        cnt = live.sum(axis=1)
        return 12 * int(cnt.sum()) + 4 * int((cnt < w).sum())

    f = e["format"]
    if f == 0:
        return 16 * e["val"].size + xy
    if f == 1:
        return 12 * e["val"].size + 8 * (n + 1) + xy
    if f == 2:
        return dia(e) + xy
    if f == 3:
        return ell(e) + xy
    if f == 4:
        return ell(e["ell"]) + 16 * e["coo"]["val"].size + xy
    return dia(e["dia"]) + (12 * e["csr"]["val"].size + 8 * (n + 1) if e["csr"]["val"].size else 0) + xy


def timed_spmv(m, x, nthreads, budget):
    per, tot = m.time_spmv(x, 1, nthreads)  # one rep (after the reference's own warm-up) sizes the run
    reps = int(max(1, min(50, budget / max(tot, 1e-6))))
    if reps > 1:
        per, tot = m.time_spmv(x, reps, nthreads)
    return tot / reps, reps


def workload(cfg):
    if cfg == 1:
        return "2-D 5-point Laplacian 1000x1000 (configs[0])", synth.laplacian_2d(1000, seed=1)
    if cfg == 2:
        return "banded n=4,000,000, 27 diagonals (configs[1])", synth.banded(4_000_000, 13, seed=2)
    if cfg == 3:
        return "R-MAT 2^22 rows, avg degree 16 (configs[2])", synth.rmat(22, 16, seed=42)
    if cfg == 5:
        return ("3-D 27-point stencil 128^3 (configs[4] scaled from 512^3: not materialisable through the "
                "CPU path)", synth.stencil_3d(128, 27, seed=5))
    raise ValueError(cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,5")
    ap.add_argument("--budget", type=float, default=1.0, help="seconds of SpMV per timing")
    a = ap.parse_args()
    ncpu = os.cpu_count() or 1
    from paper_2303_05098_b200.models import default_forest
    rf = O.RefForest(default_forest())
    cpu = None
    with open("/proc/cpuinfo") as f:
        for line in f:
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    out = {"cpu_model": cpu, "hardware_threads": ncpu, "kind": "reference",
           "build": "oracle/_ref: proj/src compiled in place, -O3 -DNDEBUG (Release flags, no -march)",
           "x": "ones (pipeline.cpp:23-25)", "configs": {}}
    for cfg in [int(c) for c in a.configs.split(",")]:
        t0 = time.perf_counter()
        name, csr = workload(cfg)
        base = O.RefMatrix.raw_coo(csr.nrows, csr.ncols, csr.coo_rows(), csr.col, csr.val)
        z = int(csr.nnz)
        del csr
        x = np.ones(base.dims[1])
        rec = {"workload": name, "nrows": base.dims[0], "ncols": base.dims[1], "nnz": z,
               "setup_s": round(time.perf_counter() - t0, 2), "formats": {}}
        csr_1t = None
        times_1t = {}
        for f in range(6):
            t1 = time.perf_counter()
            try:
                m = base.from_coo(f)
            except O.RefError as e:  # PaddingOverflow (formats.cpp:81-84, 111-112)
                rec["formats"][FMT[f]] = {"feasible": False, "why": str(e)[:120]}
                continue
            conv = time.perf_counter() - t1
            nbytes = algorithmic_bytes(m.export())
            s1, r1 = timed_spmv(m, x, 1, a.budget)
            sn, rn = timed_spmv(m, x, ncpu, a.budget)
            times_1t[f] = s1
            if f == 1:
                csr_1t = s1
            rec["formats"][FMT[f]] = {
                "feasible": True, "convert_from_coo_s": round(conv, 4), "algorithmic_bytes": int(nbytes),
                "ms_1thread": round(s1 * 1e3, 3), "reps_1thread": r1,
                "ms_all_threads": round(sn * 1e3, 3), "reps_all_threads": rn,
                "gbs_1thread": round(nbytes / s1 / 1e9, 3), "gbs_all_threads": round(nbytes / sn / 1e9, 3),
                "gflops_1thread": round(2 * z / s1 / 1e9, 3), "gflops_all_threads": round(2 * z / sn / 1e9, 3)}
            del m
        # tuner on the CSR source (the reference pipeline tunes from the loaded matrix)
        mc = base.from_coo(1)
        t2 = time.perf_counter()
        feats, _ = mc.extract_features(0.2)
        t_fe = time.perf_counter() - t2
        k = 2000
        t3 = time.perf_counter()
        for _ in range(k):
            chosen = rf.predict_forest(feats)
        t_pred = (time.perf_counter() - t3) / k
        rec["extract_features_ms"] = round(t_fe * 1e3, 3)
        rec["predict_forest_us"] = round(t_pred * 1e6, 3)
        rec["predicted"] = FMT[chosen]
        if csr_1t:
            rec["tune_cost_csr_spmv_equiv_1thread"] = round((t_fe + t_pred) / csr_1t, 3)
            opt = times_1t.get(chosen, csr_1t)
            rec["eq2_speedup_vs_csr_1000reps_1thread"] = round(1000 * csr_1t / (t_fe + t_pred + 1000 * opt), 4)
            best = min(times_1t, key=times_1t.get)
            rec["measured_optimal_1thread"] = FMT[best]
        rec["wall_s"] = round(time.perf_counter() - t0, 1)
        out["configs"][str(cfg)] = rec
        print(f"config {cfg}: {rec['wall_s']} s", file=sys.stderr, flush=True)
        del base, mc
    print(json.dumps(out))


if __name__ == "__main__":
    main()
