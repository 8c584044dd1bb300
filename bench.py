#!/usr/bin/env python3
"""Benchmark of the B200 hot path (BASELINE.json metric: SpMV GB/s & % HBM
roofline per format; tuned-vs-CSR speedup; tune overhead).

A "step" is one SpMV pass over the workload matrix (configs[1]: banded
n = 4,000,000 with 27 diagonals, fp64) in the format the on-device tuner
selects, inputs resident in HBM, L2 flushed between steps.  `value` is whole-
job GB/s of algorithmic bytes; `e2e` is the same metric through
the reference-facing call spmv(m, x) with pinned HOST x/y, H2D + D2H inside the
timed region.  N > 1 (torchrun): every rank multiplies its own copy of the
workload (independent matrices, no data-path collective) -> scaling "weak".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    "banded": "banded n=4,000,000, 27 diagonals (configs[1])",
    "laplacian": "2-D 5-point Laplacian 1000x1000 (configs[0])",
    "rmat": "R-MAT 2^22 rows, avg degree 16 (configs[2])",
}
FMT = ("COO", "CSR", "DIA", "ELL", "HYB", "HDC")
# dominant kernel per format on the workload (HDC with an empty CSR part runs the DIA kernel)
KERNEL_OF = {"COO": "coo_warp_kernel", "CSR": "csr_warp_kernel", "DIA": "dia_kernel", "ELL": "ell_kernel",
             "HYB": "ell_kernel", "HDC": "dia_kernel"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="banded", choices=sorted(CONFIGS))
    p.add_argument("--all-formats", action="store_true", default=True)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-other-configs", action="store_true",
                   help="skip the per-format lines of configs 1 and 3 (diagnostic, not the headline)")
    return p.parse_args()


def build_workload(name):
    from paper_2303_05098_b200 import synth
    if name == "banded":
        return synth.banded(4_000_000, 13, seed=2)
    if name == "laplacian":
        return synth.laplacian_2d(1000, seed=1)
    if name == "rmat":
        return synth.rmat(22, 16, seed=42)
    raise ValueError(name)


def committed_traffic(kernel, workload):
    """DRAM bytes per launch of `kernel` on `workload` from the committed ncu
    --set full capture (profiles/traffic.json, written by
    scripts/ncu_summary.py; keys "kernel@workload" or "kernel" = banded)."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None
    if f"{kernel}@{workload}" in t:
        return t[f"{kernel}@{workload}"]
    return t.get(kernel) if workload == "banded" else None


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------ reference arm

def run_reference(args, world, rank):
    """The reference's own CPU implementation (oracle/_ref) on this host."""
    if rank != 0:
        return
    import oracle as O
    csr = build_workload(args.workload)
    rows = csr.coo_rows()
    ncpu = os.cpu_count() or 1
    t0 = time.perf_counter()
    base = O.RefMatrix.raw_coo(csr.nrows, csr.ncols, rows, csr.col, csr.val)
    fmt = 2 if args.workload == "banded" else 1
    m = base.from_coo(fmt)
    build_s = time.perf_counter() - t0
    x = np.ones(csr.ncols)
    for _ in range(max(args.warmup, 1)):
        m.spmv(x, ncpu)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        m.spmv(x, ncpu)
        times.append(time.perf_counter() - t)
    import paper_2303_05098_b200 as P
    dm = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val).convert(fmt) \
        if _cuda_ok() else None
    nbytes = dm.spmv_bytes if dm is not None else _host_bytes(csr, fmt)
    ms = float(np.mean(times)) * 1e3
    gbs = nbytes / (ms * 1e-3) / 1e9
    line = {"impl": "reference", "metric": "spmv_gbs", "value": round(gbs, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": CONFIGS[args.workload], "format": FMT[fmt],
                                            "nthreads": ncpu},
            "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": ncpu, "kind": "reference",
                             "sample": f"spmv_parallel({ncpu} threads) x {args.steps} steps, "
                                       f"reference build {build_s:.1f}s"},
            "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _host_bytes(csr, fmt):
    n, z = csr.nrows, csr.nnz
    return z * 12 + (n + 1) * 8 + 16 * n


# ------------------------------------------------------------------ B200 arm

def cpu_baseline_sample(csr, fmt, budget_s=15.0):
    """The reference CPU path (oracle/_ref) timed on this host, bounded sample."""
    import oracle as O
    ncpu = os.cpu_count() or 1
    rows = csr.coo_rows()
    m = O.RefMatrix.raw_coo(csr.nrows, csr.ncols, rows, csr.col, csr.val).from_coo(fmt)
    x = np.ones(csr.ncols)
    m.spmv(x, ncpu)
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < budget_s and reps < 20:
        m.spmv(x, ncpu)
        reps += 1
    sec = (time.perf_counter() - t0) / reps
    # beside it: one thread, and the reference feature scan
    t1 = time.perf_counter()
    m.spmv(x, 1)
    sec1 = time.perf_counter() - t1
    t2 = time.perf_counter()
    m.extract_features(0.2)
    fe = time.perf_counter() - t2
    return sec, reps, ncpu, {"single_thread_s": sec1, "extract_features_s": fe}


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2303_05098_b200 as P
    from paper_2303_05098_b200 import _capi

    P.set_device(local)
    csr = build_workload(args.workload)
    base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)

    # a dedicated (non-legacy) stream: kernels and timing events share it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    assert sptr != 0
    x = torch.ones(csr.ncols, dtype=torch.float64, device="cuda")
    y = torch.empty(csr.nrows, dtype=torch.float64, device="cuda")
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    flush = torch.empty(max(2 * l2, 1 << 28) // 4, dtype=torch.float32, device="cuda")
    peak, peak_kind = peaks()

    def needs_flush(m):
        # matrices >= 4x L2 stream through it every step (nothing of the
        # previous step survives); smaller ones (config 1) get a 2x-L2 write
        return m.spmv_bytes < 4 * l2

    def time_format(m, steps, warmup, count=False):
        fl = needs_flush(m)
        for _ in range(warmup):
            if fl:
                flush.fill_(1.0)
            m.spmv_device(x.data_ptr(), y.data_ptr(), sptr)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        torch.cuda.synchronize()
        n0 = _capi.lib().so_kernel_launches()
        for a, b in ev:
            if fl:
                flush.fill_(1.0)
            a.record(stream)
            m.spmv_device(x.data_ptr(), y.data_ptr(), sptr)
            b.record(stream)
        torch.cuda.synchronize()
        times = [a.elapsed_time(b) * 1e-3 for a, b in ev]
        return (times, _capi.lib().so_kernel_launches() - n0) if count else times

    # ---- per-format table (formats that fit the padding cap) -----------------
    per_format = {}
    mats = {}
    for f in range(6):
        try:
            mats[f] = base.convert(f)
        except P.PaddingOverflow:
            per_format[FMT[f]] = {"feasible": False}
            continue
        t = time_format(mats[f], max(10, args.steps // 2), 3)
        nbytes = mats[f].spmv_bytes
        sec = float(np.mean(t))
        per_format[FMT[f]] = {"feasible": True, "ms": round(sec * 1e3, 4),
                              "gbs": round(nbytes / sec / 1e9, 1),
                              "frac": round(nbytes / sec / 1e9 / peak, 3), "bytes": nbytes}

    # ---- configs 1 and 3, per format (diagnostic lines beside the headline) ---
    other = {}
    if not args.no_other_configs and rank == 0:
        from paper_2303_05098_b200 import synth, synth_dev
        lap = synth.laplacian_2d(1000, seed=1)
        work = {"config1 laplacian 1000^2 (host generator, seed 1)":
                P.DeviceMatrix.csr(lap.nrows, lap.ncols, lap.row_ptr, lap.col, lap.val),
                "config3 rmat 2^22 d16 (device generator, seed 42)":
                synth_dev.rmat(1 << 22, 16, 42).to_device_matrix()}
        # HYB's favourable shape: config 3 is gather-bound for
        # every format, so HYB is also reported on rows that fill
        # its ELL part with 1 % of rows overflowing into the COO part
        hyb = synth.hyb_skewed(4_000_000, 16, 160, 100, seed=6)
        work["hyb-favourable n=4M, 16-entry rows, every 100th row 160 (K_H=18, COO part 8 %; host generator, seed 6)"] = \
            P.DeviceMatrix.csr(hyb.nrows, hyb.ncols, hyb.row_ptr, hyb.col, hyb.val)
        del hyb, lap
        for wname, wbase in work.items():
            xo = torch.ones(wbase.ncols, dtype=torch.float64, device="cuda")
            yo = torch.empty(wbase.nrows, dtype=torch.float64, device="cuda")
            row = {}
            for f in range(6):
                try:
                    mo = wbase.convert(f)
                except P.PaddingOverflow:
                    row[FMT[f]] = "infeasible"
                    continue
                # small matrices: rotate over enough copies (matrix and x) that
                # every step reads cold inputs -- "inputs larger than L2"
                # without the dirty-line write-back a write flush leaves behind
                ncopy = int(np.ceil(3 * l2 / max(mo.spmv_bytes, 1))) + 1 if needs_flush(mo) else 1
                mats_o = [mo] + [mo.convert(f) for _ in range(ncopy - 1)]
                xs_o = [xo] + [torch.ones_like(xo) for _ in range(ncopy - 1)]
                # steps enqueued back to back (events on the launching stream,
                # one sync at the end), as in time_format
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(23)]
                # one untimed multiply per copy: a matrix's first multiply may
                # profile it (COO: coo_max_gap + a host read, cached after)
                for k in range(ncopy):
                    mats_o[k].spmv_device(xs_o[k].data_ptr(), yo.data_ptr(), sptr)
                torch.cuda.synchronize()
                for r, (a_, b_) in enumerate(evs):
                    k = r % ncopy
                    a_.record(stream)
                    mats_o[k].spmv_device(xs_o[k].data_ptr(), yo.data_ptr(), sptr)
                    b_.record(stream)
                torch.cuda.synchronize()
                ts = [a_.elapsed_time(b_) * 1e-3 for a_, b_ in evs[3:]]
                fl = ncopy > 1
                del mats_o, xs_o
                sec_o = float(np.mean(ts))
                row[FMT[f]] = {"ms": round(sec_o * 1e3, 4), "gbs": round(mo.spmv_bytes / sec_o / 1e9, 1),
                               "frac": round(mo.spmv_bytes / sec_o / 1e9 / peak, 3),
                               "l2": f"rotating {ncopy} copies (cold inputs)" if fl else "larger than L2"}
                del mo
            other[wname] = row
            del wbase, xo, yo
        torch.cuda.empty_cache()

    # ---- tuner: on-device features + predict (measured-optimal label model) ---
    best = min((f for f in mats), key=lambda f: per_format[FMT[f]]["ms"])
    tuned = best
    tune = None
    try:
        from paper_2303_05098_b200.models import default_forest
        forest = P.DeviceForest(default_forest())
        o = P.tune_ml(base, forest)
        tuned = int(o.chosen)
        outs = [P.tune_ml(base, forest) for _ in range(5)]
        t_fe = float(np.median([q.feature_time_seconds for q in outs]))
        t_pr = float(np.median([q.predict_time_seconds for q in outs]))
        t_csr = per_format["CSR"]["ms"] * 1e-3
        tune = {"chosen": FMT[tuned], "measured_optimal": FMT[best], "t_fe_ms": round(t_fe * 1e3, 4),
                "t_pred_ms": round(t_pr * 1e3, 4),
                "overhead_csr_spmv_equiv": round((t_fe + t_pr) / t_csr, 3),
                # pipeline.cpp:298-302: T_CSR / (T_FE + T_PRED + T_OPT), reps = 1000 multiplies
                "speedup_vs_csr_reps1000": round(1000 * t_csr / (t_fe + t_pr + 1000 * per_format[FMT[tuned]]["ms"] * 1e-3),
                                                 3)}
    except Exception as e:  # model not available yet
        tune = {"error": str(e)[:200], "chosen": FMT[tuned], "measured_optimal": FMT[best]}
    m = mats[tuned]
    nbytes = m.spmv_bytes

    # ---- headline: timed steps ----------------------------------------------
    clocks = ClockSampler(local)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t, launches = time_format(m, args.steps, max(args.warmup, 3), count=True)
    clk = clocks.stop()
    sec = float(np.mean(t))
    tmax = torch.tensor([sec], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
    sec = float(tmax.item())
    value = world * nbytes / sec / 1e9

    # ---- e2e through spmv(m, x): pinned host x/y, H2D + kernel + D2H ----------
    xh = torch.ones(csr.ncols, dtype=torch.float64).pin_memory()
    yh = torch.empty(csr.nrows, dtype=torch.float64).pin_memory()
    xn, yn = xh.numpy(), yh.numpy()
    for _ in range(3):
        m.spmv_into(xn, yn)
    e2e_t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        m.spmv_into(xn, yn)
        e2e_t.append(time.perf_counter() - t0)
    e2e_sec = float(np.mean(e2e_t))
    et = torch.tensor([e2e_sec], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
    e2e_sec = float(et.item())

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cs, reps, cores, extra = cpu_baseline_sample(csr, tuned)
                cpu = {"value": round(nbytes / cs / 1e9, 3), "unit": "GB/s", "cores": cores,
                       "kind": "reference",
                       "sample": f"reference spmv_parallel({cores}) on the same {FMT[tuned]} matrix, "
                                 f"{reps} reps",
                       "single_thread_value": round(nbytes / extra["single_thread_s"] / 1e9, 3),
                       "extract_features_ms": round(extra["extract_features_s"] * 1e3, 2)}
            except Exception as e:
                cpu = {"error": str(e)[:200]}
        line = {
            "metric": "spmv_gbs", "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": CONFIGS[args.workload], "format": FMT[tuned],
                       "l2": ("flushed between steps (write of 2x L2)" if needs_flush(m) else
                              f"inputs larger than L2 ({nbytes / l2:.1f}x the {l2 >> 20} MB L2), no flush"),
                       "nnz": csr.nnz,
                       "nrows": csr.nrows, "parallelism": f"replicas x{world}"},
            "roofline": {"bound": "hbm", "achieved": round(nbytes / sec / 1e9, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(nbytes / sec / 1e9 / peak, 4),
                         "traffic": committed_traffic(KERNEL_OF[FMT[tuned]], args.workload), "algorithmic_bytes": nbytes,
                         "kernel": KERNEL_OF[FMT[tuned]], "peak_kind": peak_kind},
            "e2e": {"value": round(world * nbytes / e2e_sec / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * csr.ncols, "d2h_bytes_per_step": 8 * csr.nrows},
            "gpu_launches": launches,
            "clocks": clk, "cpu_baseline": cpu, "formats": per_format, "tune": tune,
            "other_configs": other,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
