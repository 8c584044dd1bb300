#!/usr/bin/env python3
"""Benchmark of the B200 hot path (BASELINE.json metric: SpMV GB/s & % HBM
roofline per format; tuned-vs-CSR speedup; tune overhead).

N = 1 (headline): a "step" is one SpMV pass over the config-2 matrix (banded
n = 4,000,000 with 27 diagonals, fp64; BASELINE.json configs[1]) in the format
the on-device tuner selects, inputs resident in HBM.  `value` is GB/s of
algorithmic bytes; `e2e` is the same metric through the
reference-facing call spmv(m, x) (so_spmv) with pinned host x/y -- H2D + D2H
inside the timed region -- with `e2e_pageable` (numpy buffers: the library
stages them through pinned memory with host threads) and `e2e_cpp_api`
(sparseoracle::spmv returning a fresh std::vector) beside it.  Also in the line:
per-format tables for configs 1-3, the tuner on config 2 and on a held-out
100-matrix slice of the config-4 batch (tuning cost in CSR-SpMV equivalents,
device and host wall clock; Eq. 2 speedup at 1000 repetitions), config 5
(27-point stencil 512^3) iterated on one GPU, and the reference CPU path.

N > 1 (torchrun, one process per GPU): config 5 row-partitioned over the
ranks -- 27-point stencil 512^3, DIA, x halos pushed into the neighbours'
windows by the multiply itself over NVLink peer memory (so_dist_*), strong
scaling; `value` = whole-job GB/s (all ranks' bytes / max-over-ranks time),
plus a config-4 shard throughput (matrices/s, LPT-sharded, no collective on
the data path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import math
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
CONFIG5 = "3-D 27-point stencil 512^3 (134M rows, 3.6e9 nnz), row-partitioned iterated SpMV (configs[4])"
FMT = ("COO", "CSR", "DIA", "ELL", "HYB", "HDC")
# dominant kernel per format on the workload (HDC with an empty CSR part runs the DIA kernel)
KERNEL_OF = {"COO": "coo_warp_kernel", "CSR": "csr_warp_kernel", "DIA": "dia_kernel", "ELL": "ell_kernel",
             "HYB": "ell_kernel", "HDC": "dia_kernel"}
G5 = 512  # config 5 grid


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="banded", choices=sorted(CONFIGS))
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-other-configs", action="store_true",
                   help="skip the per-format lines of configs 1 and 3 (diagnostic, not the headline)")
    p.add_argument("--no-config4", action="store_true", help="skip the config-4 slice")
    p.add_argument("--no-config5", action="store_true", help="skip config 5 at N=1")
    p.add_argument("--config4-count", type=int, default=100)
    p.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                   help="N>1 halo exchange: fused peer-memory push (default) or NCCL isend/irecv")
    return p.parse_args()


def _synth():
    """paper_2303_05098_b200/synth.py loaded by path: the reference arm must not
    import (and so map) the product package."""
    spec = importlib.util.spec_from_file_location("_bench_synth", os.path.join(REPO, "paper_2303_05098_b200",
                                                                                "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_bench_synth"] = mod  # dataclasses look their module up
    spec.loader.exec_module(mod)
    return mod


def build_workload(name):
    synth = _synth()
    if name == "banded":
        return synth.banded(4_000_000, 13, seed=2)
    if name == "laplacian":
        return synth.laplacian_2d(1000, seed=1)
    if name == "rmat":
        return synth.rmat(22, 16, seed=42)
    raise ValueError(name)


def workload_format(name):
    return 2 if name == "banded" else 1  # DIA on the banded matrix (the tuner's choice), else CSR


def common_config(name, nrows, nnz, world):
    """The `config` dict both arms print (identical keys and values)."""
    fmt = FMT[workload_format(name)]
    return {"workload": CONFIGS[name], "format": fmt, "nnz": int(nnz), "nrows": int(nrows),
            "parallelism": "single device" if world == 1 else f"replicas x{world}"}


def config5_config(world):
    n = G5 ** 3
    return {"workload": CONFIG5, "format": "DIA", "nnz": (3 * G5 - 2) ** 3, "nrows": n,
            "parallelism": f"row partition x{world}, halo {G5 * G5 + G5 + 1} rows per side"}


def host_algorithmic_bytes(csr, fmt):
    """so_spmv_bytes of DESIGN.md §4 computed from host arrays (pure Python):
    DIA 8*sum(clipped diagonal lengths) + 8*D + x + y; CSR 12 z + 8 (n+1) + x + y."""
    n, m = csr.nrows, csr.ncols
    if fmt == 2:
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(csr.row_ptr))
        offs = np.unique(csr.col - rows)
        cells = sum(max(0, min(n, m - int(o)) - max(0, -int(o))) for o in offs)
        return 8 * cells + 8 * offs.size + 8 * m + 8 * n
    return 12 * csr.nnz + 8 * (n + 1) + 8 * m + 8 * n


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    NVML (pynvml, microseconds per query) polled every ~0.5 ms from a thread,
    so even a few-millisecond timed region gets samples inside it; the first
    sample is taken before start() returns.  Falls back to nvidia-smi (tens
    of ms per query) when NVML is unavailable.  The NVML device is the CUDA
    device's PCI bus id (CUDA and NVML ordinals differ under
    CUDA_VISIBLE_DEVICES)."""

    NAMES = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
             ("sw_power_cap", 0x4))

    def __init__(self, index=0):
        self.index = index
        self.samples = []  # (sm_mhz, sm_max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        self.source = "nvidia-smi"
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            try:
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._nvml = (pynvml, h)
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        pynvml, h = self._nvml
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        try:
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.samples.append((float(sm), float(mx), int(rs)))

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                              "--format=csv,noheader,nounits"], capture_output=True,
                             text=True, timeout=5).stdout.strip()
        if out:
            f = [v.strip() for v in out.split(",")]
            if f[0].replace(".", "").isdigit() and f[1].replace(".", "").isdigit():
                mask = sum(bit for (_, bit), v in zip(self.NAMES, f[2:]) if v.lower().startswith("active"))
                self.samples.append((float(f[0]), float(f[1]), mask))

    def _sample(self):
        try:
            self._sample_nvml() if self._nvml else self._sample_smi()
        except Exception:
            pass

    def start(self):
        self._sample()  # one sample before the timed region starts
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.0005 if self._nvml else 0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        self._sample()  # and one right after
        sm = [v[0] for v in self.samples]
        mx = [v[1] for v in self.samples]
        reasons = sorted({name for v in self.samples for name, bit in self.NAMES if v[2] & bit})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------ reference arm

def stencil27_slice_coo(g, r0, r1, seed=5):
    """Rows [r0, r1) of the 27-point stencil on a g^3 grid as (rows, cols,
    vals), global column indices -- a bounded host sample of config 5."""
    i = np.arange(r0, r1, dtype=np.int64)
    z, rem = np.divmod(i, g * g)
    y, x = np.divmod(rem, g)
    rows, cols = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((z + dz >= 0) & (z + dz < g) & (y + dy >= 0) & (y + dy < g) & (x + dx >= 0) & (x + dx < g))
                rows.append(i[ok])
                cols.append((i + dz * g * g + dy * g + dx)[ok])
    r, c = np.concatenate(rows), np.concatenate(cols)
    order = np.lexsort((c, r))
    r, c = r[order], c[order]
    v = np.random.default_rng(seed).uniform(0.5, 2.0, r.size)
    return r, c, v


def run_reference(args, world, rank):
    """The reference's own CPU implementation (oracle/_ref: proj/src compiled
    in place, unmodified) timed with its own time_spmv (spmv.cpp:221-246) on
    all host threads, on this arm's workload, config, metric and unit.  The
    product package is never imported here."""
    if rank != 0:
        return
    import oracle as O
    ncpu = os.cpu_count() or 1
    t0 = time.perf_counter()
    if world == 1:
        csr = build_workload(args.workload)
        fmt = workload_format(args.workload)
        rows = np.repeat(np.arange(csr.nrows, dtype=np.int64), np.diff(csr.row_ptr))
        m = O.RefMatrix.raw_coo(csr.nrows, csr.ncols, rows, csr.col, csr.val).from_coo(fmt)
        nbytes = host_algorithmic_bytes(csr, fmt)
        config = common_config(args.workload, csr.nrows, csr.nnz, world)
        x = np.ones(csr.ncols)
        sample = f"time_spmv(1 rep, {ncpu} threads) per step on the full {FMT[fmt]} matrix"
        del csr, rows
    else:
        # config 5 is not materialisable through the CPU path (SURVEY §8d,
        # BASELINE.md §4): a 2^21-row slab of the same 512^3 stencil
        g, n = G5, G5 ** 3
        r0, r1 = n // 2, n // 2 + (1 << 21)
        h = g * g + g + 1
        r, c, v = stencil27_slice_coo(g, r0, r1)
        w0 = r0 - h
        m = O.RefMatrix.raw_coo(r1 - r0, 2 * h + (r1 - r0), r - r0, c - w0, v).from_coo(2)
        d = np.unique(c - r)
        nbytes = 8 * r.size + 8 * d.size + 8 * (2 * h + r1 - r0) + 8 * (r1 - r0)
        config = config5_config(world)
        x = np.ones(2 * h + (r1 - r0))
        sample = (f"time_spmv(1 rep, {ncpu} threads) per step on rows [{r0}, {r1}) of the 512^3 stencil "
                  f"(DIA, {r.size} nnz): the whole matrix does not fit the CPU path")
    build_s = time.perf_counter() - t0
    for _ in range(max(args.warmup, 1)):
        m.time_spmv(x, 1, ncpu)
    times = []
    for _ in range(args.steps):
        per, tot = m.time_spmv(x, 1, ncpu)
        times.append(tot)
    sec = float(np.mean(times))
    gbs = nbytes / sec / 1e9
    line = {"impl": "reference", "metric": "spmv_gbs", "value": round(gbs, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 4),
            "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config,
            "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": ncpu, "kind": "reference",
                             "sample": sample + f"; reference build + conversion {build_s:.1f}s",
                             "cpu_model": cpu_model()},
            "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm

def cpu_baseline_sample(csr, fmt, budget_s=12.0):
    """The reference CPU path (oracle/_ref) timed on this host with its own
    time_spmv, bounded sample, plus one thread, extract_features and
    predict_forest beside it."""
    import oracle as O
    ncpu = os.cpu_count() or 1
    rows = csr.coo_rows()
    t0 = time.perf_counter()
    base = O.RefMatrix.raw_coo(csr.nrows, csr.ncols, rows, csr.col, csr.val)
    m = base.from_coo(fmt)
    t_convert = time.perf_counter() - t0
    x = np.ones(csr.ncols)
    m.time_spmv(x, 1, ncpu)
    reps = 0
    tot = 0.0
    while tot < budget_s and reps < 20:
        _, t = m.time_spmv(x, 1, ncpu)
        tot += t
        reps += 1
    sec = tot / reps
    _, sec1 = m.time_spmv(x, 1, 1)
    t2 = time.perf_counter()
    m.extract_features(0.2)
    fe = time.perf_counter() - t2
    pred_us = None
    try:
        rf = O.RefForest(forest_ff())  # the reference's predict_forest on the shipped forest
        row = np.array(m.extract_features(0.2)[0])
        t3 = time.perf_counter()
        for _ in range(2000):
            rf.predict_forest(row)
        pred_us = (time.perf_counter() - t3) / 2000 * 1e6  # includes the ctypes call
    except Exception:
        pass
    return {"sec": sec, "reps": reps, "cores": ncpu, "single_thread_s": sec1, "extract_features_s": fe,
            "convert_s": t_convert, "predict_forest_us": pred_us}


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch

    ndev = max(torch.cuda.device_count(), 1)
    dev = local % ndev  # ranks sharing a GPU (tests) still work
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if ndev >= world else "gloo",
                                device_id=torch.device("cuda", dev) if ndev >= world else None)
    import paper_2303_05098_b200 as P

    P.set_device(dev)
    if world > 1:
        return run_partitioned(args, world, rank, dev)
    return run_single(args, dev)


def time_steps(m, x, y, stream, steps, warmup, flush=None, count=False):
    """`steps` multiplies back to back, each bracketed by CUDA events on the
    launching stream (optionally behind an L2-flushing write)."""
    import torch
    from paper_2303_05098_b200 import _capi
    for _ in range(warmup):
        if flush is not None:
            flush.fill_(1.0)
        m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    n0 = _capi.lib().so_kernel_launches()
    for a, b in ev:
        if flush is not None:
            flush.fill_(1.0)
        a.record(stream)
        m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
        b.record(stream)
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) * 1e-3 for a, b in ev]
    return (times, _capi.lib().so_kernel_launches() - n0) if count else times


def run_single(args, dev):
    import torch
    import paper_2303_05098_b200 as P
    from paper_2303_05098_b200 import synth

    csr = build_workload(args.workload)
    base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    x = torch.ones(csr.ncols, dtype=torch.float64, device="cuda")
    y = torch.empty(csr.nrows, dtype=torch.float64, device="cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(max(2 * l2, 1 << 28) // 4, dtype=torch.float32, device="cuda")
    peak, peak_kind = peaks()

    def flush_for(m):
        # matrices >= 4x L2 stream through it every step (nothing of the
        # previous step survives); smaller ones (config 1) get a 2x-L2 write
        return flush_buf if m.spmv_bytes < 4 * l2 else None

    # ---- per-format table (formats that fit the padding cap) -----------------
    per_format, mats = {}, {}
    for f in range(6):
        try:
            mats[f] = base.convert(f)
        except P.PaddingOverflow:
            per_format[FMT[f]] = {"feasible": False}
            continue
        t = time_steps(mats[f], x, y, stream, max(10, args.steps // 2), 3, flush_for(mats[f]))
        nbytes = mats[f].spmv_bytes
        sec = float(np.mean(t))
        per_format[FMT[f]] = {"feasible": True, "ms": round(sec * 1e3, 4), "gbs": round(nbytes / sec / 1e9, 1),
                              "frac": round(nbytes / sec / 1e9 / peak, 3), "bytes": nbytes}

    other = {} if args.no_other_configs else other_configs(P, synth, stream, l2, peak)

    # ---- tuner on the workload: device intervals and host wall clock ----------
    best = min((f for f in mats), key=lambda f: (per_format[FMT[f]]["ms"], f))
    tuned, tune = best, None
    try:
        from paper_2303_05098_b200.models import default_forest
        forest = P.DeviceForest(default_forest())
        tuned = int(P.tune_ml(base, forest).chosen)
        outs = [P.tune_ml(base, forest) for _ in range(7)]
        t_fe = float(np.median([q.feature_time_seconds for q in outs]))
        t_pr = float(np.median([q.predict_time_seconds for q in outs]))
        t_wall = float(np.median([q.wall_time_seconds for q in outs]))  # host clock inside so_tune_ml
        t_csr = per_format["CSR"]["ms"] * 1e-3
        t_opt = per_format[FMT[tuned]]["ms"] * 1e-3
        tune = {"chosen": FMT[tuned], "measured_optimal": FMT[best], "t_fe_ms": round(t_fe * 1e3, 4),
                "t_pred_ms": round(t_pr * 1e3, 4), "t_wall_ms": round(t_wall * 1e3, 4),
                # pipeline.cpp:300-302: (T_FE + T_PRED) / (T_CSR per rep)
                "overhead_csr_spmv_equiv": round((t_fe + t_pr) / t_csr, 3),
                "overhead_csr_spmv_equiv_wall": round(t_wall / t_csr, 3),
                # pipeline.cpp:298-299: T_CSR / (T_FE + T_PRED + T_OPT), reps = 1000 multiplies
                "speedup_vs_csr_reps1000": round(1000 * t_csr / (t_fe + t_pr + 1000 * t_opt), 3),
                "speedup_vs_csr_reps1000_wall": round(1000 * t_csr / (t_wall + 1000 * t_opt), 3)}
    except Exception as e:  # model not available
        tune = {"error": str(e)[:200], "chosen": FMT[tuned], "measured_optimal": FMT[best]}
    m = mats[tuned]
    nbytes = m.spmv_bytes
    for f in list(mats):
        if f != tuned:
            del mats[f]

    # ---- headline: timed steps ----------------------------------------------
    clocks = ClockSampler(dev)
    torch.cuda.synchronize()
    clocks.start()
    t, launches = time_steps(m, x, y, stream, args.steps, max(args.warmup, 3), flush_for(m), count=True)
    clk = clocks.stop()
    sec = float(np.mean(t))
    value = nbytes / sec / 1e9

    # ---- e2e through spmv(m, x): host x/y, H2D + kernel + D2H per step --------
    e2e = e2e_numbers(m, csr, args.steps, nbytes)
    del flush_buf, x, y

    cfg4 = None if args.no_config4 else config4_slice(P, stream, args.config4_count, forest_ff())
    cfg5 = None if args.no_config5 else config5_single(P, stream, peak)

    cpu = None
    if not args.no_cpu_baseline:
        try:
            c = cpu_baseline_sample(csr, tuned)
            cpu = {"value": round(nbytes / c["sec"] / 1e9, 3), "unit": "GB/s", "cores": c["cores"],
                   "kind": "reference", "cpu_model": cpu_model(),
                   "sample": f"reference time_spmv(1 rep, {c['cores']} threads) x {c['reps']} on the same "
                             f"{FMT[tuned]} matrix",
                   "single_thread_value": round(nbytes / c["single_thread_s"] / 1e9, 3),
                   "extract_features_ms": round(c["extract_features_s"] * 1e3, 2),
                   "convert_from_coo_s": round(c["convert_s"], 3),
                   "predict_forest_us": None if c["predict_forest_us"] is None else round(c["predict_forest_us"], 3)}
        except Exception as e:
            cpu = {"error": str(e)[:200]}
    line = {
        "metric": "spmv_gbs", "value": round(value, 2), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": common_config(args.workload, csr.nrows, csr.nnz, 1),
        "l2_policy": ("flushed between steps (write of 2x L2)" if flush_for(m) is not None else
                      f"inputs larger than L2 ({nbytes / l2:.1f}x the {l2 >> 20} MB L2), no flush"),
        "roofline": {"bound": "hbm", "achieved": round(value, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(value / peak, 4),
                     "traffic": committed_traffic(KERNEL_OF[FMT[tuned]], args.workload),
                     "algorithmic_bytes": nbytes, "kernel": KERNEL_OF[FMT[tuned]], "peak_kind": peak_kind},
        "e2e": e2e.pop("pinned"),
        **e2e,
        "gpu_launches": launches,
        "clocks": clk, "cpu_baseline": cpu, "formats": per_format, "tune": tune,
        "config4_slice": cfg4, "config5_n1": cfg5, "other_configs": other,
    }
    print(json.dumps(line), flush=True)


def forest_ff():
    from paper_2303_05098_b200.models import default_forest
    return default_forest()


def e2e_numbers(m, csr, steps, nbytes):
    """spmv(m, x) with host buffers: pageable numpy (the reference API's own
    case -- so_spmv stages through pinned memory with host threads), pinned
    torch buffers, and the C++ drop-in call itself (scripts/e2e_api.cpp:
    sparseoracle::spmv returning a fresh std::vector)."""
    import torch
    out = {}
    xh = np.ones(csr.ncols)
    yh = np.empty(csr.nrows)
    xp = torch.ones(csr.ncols, dtype=torch.float64).pin_memory()
    yp = torch.empty(csr.nrows, dtype=torch.float64).pin_memory()
    for key, (xx, yy) in (("e2e_pageable", (xh, yh)), ("pinned", (xp.numpy(), yp.numpy()))):
        for _ in range(3):
            m.spmv_into(xx, yy)
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            m.spmv_into(xx, yy)
            ts.append(time.perf_counter() - t0)
        sec = float(np.mean(ts))
        out[key] = {"value": round(nbytes / sec / 1e9, 2), "unit": "GB/s", "ms": round(sec * 1e3, 4),
                    "h2d_bytes_per_step": 8 * csr.ncols, "d2h_bytes_per_step": 8 * csr.nrows,
                    "host_buffers": "pageable (numpy)" if key == "e2e_pageable" else "pinned (torch)",
                    "call": "so_spmv(m, x, n, y) -- what sparseoracle::spmv(m, x) calls"}
    exe = os.path.join(REPO, "build", "e2e_api")
    if os.path.exists(exe):
        try:
            r = subprocess.run([exe, str(min(steps, 20)), "3"], capture_output=True, text=True, timeout=300)
            d = json.loads(r.stdout.strip().splitlines()[-1])
            out["e2e_cpp_api"] = {"value": d["gbs_mean"], "unit": "GB/s", "ms": d["ms_mean"],
                                  "h2d_bytes_per_step": d["h2d_bytes_per_step"],
                                  "d2h_bytes_per_step": d["d2h_bytes_per_step"], "call": d["api"],
                                  "zero_fill_ms": d.get("zero_fill_ms_median")}
        except Exception as e:
            out["e2e_cpp_api"] = {"error": str(e)[:200]}
    return out


def other_configs(P, synth, stream, l2, peak):
    """Configs 1 and 3 (and HYB's favourable shape) per format, device
    resident, steps back to back; small matrices rotate cold copies."""
    import torch
    lap = synth.laplacian_2d(1000, seed=1)
    rm = synth.rmat(22, 16, seed=42)  # the matrix tests/test_gpu_full_size.py checks against the oracle
    work = {"config1 laplacian 1000^2 (host generator, seed 1)":
            P.DeviceMatrix.csr(lap.nrows, lap.ncols, lap.row_ptr, lap.col, lap.val),
            "config3 rmat 2^22 d16 (synth.rmat, seed 42)":
            P.DeviceMatrix.csr(rm.nrows, rm.ncols, rm.row_ptr, rm.col, rm.val)}
    # HYB's favourable shape: config 3 is gather-bound for every
    # format, so HYB is also reported on rows that fill its ELL
    # part with 1 % of rows overflowing into the COO part
    hyb = synth.hyb_skewed(4_000_000, 16, 160, 100, seed=6)
    work["hyb-favourable n=4M, 16-entry rows, every 100th row 160 (K_H=18, COO part 8 %; host generator, seed 6)"] = \
        P.DeviceMatrix.csr(hyb.nrows, hyb.ncols, hyb.row_ptr, hyb.col, hyb.val)
    del hyb, lap, rm
    other = {}
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
            # small matrices: rotate over enough copies (matrix and x) that every
            # step reads cold inputs -- "inputs larger than L2" without the
            # dirty-line write-back a write flush leaves behind
            ncopy = int(np.ceil(3 * l2 / max(mo.spmv_bytes, 1))) + 1 if mo.spmv_bytes < 4 * l2 else 1
            mats_o = [mo] + [mo.convert(f) for _ in range(ncopy - 1)]
            xs_o = [xo] + [torch.ones_like(xo) for _ in range(ncopy - 1)]
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(23)]
            for k in range(ncopy):  # first multiply may profile the matrix (COO), untimed
                mats_o[k].spmv_device(xs_o[k].data_ptr(), yo.data_ptr(), stream.cuda_stream)
            torch.cuda.synchronize()
            for r, (a_, b_) in enumerate(evs):
                k = r % ncopy
                a_.record(stream)
                mats_o[k].spmv_device(xs_o[k].data_ptr(), yo.data_ptr(), stream.cuda_stream)
                b_.record(stream)
            torch.cuda.synchronize()
            ts = [a_.elapsed_time(b_) * 1e-3 for a_, b_ in evs[3:]]
            del mats_o, xs_o
            sec_o = float(np.mean(ts))
            row[FMT[f]] = {"ms": round(sec_o * 1e3, 4), "gbs": round(mo.spmv_bytes / sec_o / 1e9, 1),
                           "frac": round(mo.spmv_bytes / sec_o / 1e9 / peak, 3),
                           "l2": f"rotating {ncopy} copies (cold inputs)" if ncopy > 1 else "larger than L2"}
            del mo
        other[wname] = row
        del wbase, xo, yo
    torch.cuda.empty_cache()
    return other


# ----------------------------------------------------------- config 4 slice

def held_out_ids(count):
    with open(os.path.join(REPO, "profiles", "config4_split_r02.json")) as f:
        ids = json.load(f)["test_ids"]
    return ids[:count]


def profile_one(P, spec, forest, stream, reps=10):
    """One corpus matrix: every feasible format timed (time_spmv semantics:
    reps back-to-back multiplies after a warm-up, total time; label = argmin,
    ties to the lowest id, pipeline.cpp:85-104), then tune_ml (device T_FE,
    T_PRED and the host wall clock of the call)."""
    import torch
    from paper_2303_05098_b200 import synth_dev
    dc = synth_dev.build(spec)
    base = dc.to_device_matrix()
    del dc
    x = torch.ones(base.ncols, dtype=torch.float64, device="cuda")
    y = torch.empty(base.nrows, dtype=torch.float64, device="cuda")
    tot, mats = {}, {}
    for f in range(6):
        try:
            mats[f] = base.convert(f)
        except P.PaddingOverflow:
            continue
        tot[f] = float(np.sum(time_steps(mats[f], x, y, stream, reps, 1)))
    tw = P.kernel_twins(mats)
    del mats
    P.tune_ml(base, forest)  # first call builds the tune graph
    outs = [P.tune_ml(base, forest) for _ in range(3)]
    o = outs[-1]
    return {"id": spec["id"], "family": spec["family"], "n": base.nrows, "nnz": base.nnz(),
            "t": tot, "label": min(tot, key=lambda f: (tot[f], f)), "chosen": int(o.chosen), "twins": tw,
            "t_fe": float(np.median([q.feature_time_seconds for q in outs])),
            "t_pred": float(np.median([q.predict_time_seconds for q in outs])),
            "t_wall": float(np.median([q.wall_time_seconds for q in outs])), "reps": reps}


def summarise_config4(rows, elapsed, world):
    lab = np.array([r["label"] for r in rows])
    ch = np.array([r["chosen"] for r in rows])
    t_ch = np.array([r["t"][r["chosen"]] for r in rows]) / rows[0]["reps"]
    t_opt = np.array([r["t"][r["label"]] for r in rows]) / rows[0]["reps"]
    t_csr = np.array([r["t"][1] for r in rows]) / rows[0]["reps"]
    tfe = np.array([r["t_fe"] for r in rows])
    tpr = np.array([r["t_pred"] for r in rows])
    twall = np.array([r["t_wall"] for r in rows])
    # kernel-identical twins collapse into one class (the measured "optimum"
    # between two identical kernels is timing noise)
    from paper_2303_05098_b200 import collapse_label
    lab_c = np.array([collapse_label(r["label"], r["twins"]) for r in rows])
    ch_c = np.array([collapse_label(r["chosen"], r["twins"]) for r in rows])
    recalls = [float((ch_c[lab_c == c] == c).mean()) for c in range(6) if (lab_c == c).any()]
    cost = (tfe + tpr) / t_csr
    cost_w = twall / t_csr
    sp = 1000 * t_csr / (tfe + tpr + 1000 * t_ch)
    sp_w = 1000 * t_csr / (twall + 1000 * t_ch)
    q = lambda a: {"mean": round(float(a.mean()), 3), "median": round(float(np.median(a)), 3),  # noqa: E731
                   "max": round(float(a.max()), 3)}
    gm = lambda a: round(float(np.exp(np.log(a).mean())), 4)  # noqa: E731
    return {
        "matrices": len(rows), "families": {f: int(sum(r["family"] == f for r in rows))
                                            for f in ("stencil", "banded", "uniform", "powerlaw")},
        "source": "held-out ids of profiles/config4_split_r02.json (device generators, synth_dev.corpus_spec)",
        "model": "paper_2303_05098_b200/models/b200_forest.txt",
        "accuracy": round(float((ch == lab).mean()), 4),
        "accuracy_twins_collapsed": round(float((ch_c == lab_c).mean()), 4),
        "balanced_accuracy_twins_collapsed": round(float(np.mean(recalls)), 4),
        "within_2pct_of_optimal": round(float((t_ch <= 1.02 * t_opt).mean()), 4),
        "within_5pct_of_optimal": round(float((t_ch <= 1.05 * t_opt).mean()), 4),
        "tuning_cost_csr_spmv_equiv_device": q(cost),
        "tuning_cost_csr_spmv_equiv_wall": q(cost_w),
        "eq2_speedup_vs_csr_1000reps_geomean_device": gm(sp),
        "eq2_speedup_vs_csr_1000reps_geomean_wall": gm(sp_w),
        "tuned_spmv_speedup_vs_csr_geomean": gm(t_csr / t_ch),
        "optimal_spmv_speedup_vs_csr_geomean": gm(t_csr / t_opt),
        "elapsed_s": round(elapsed, 2), "matrices_per_s": round(len(rows) / elapsed, 3), "n_gpus": world,
    }


def config4_slice(P, stream, count, ff, world=1, rank=0):
    import torch
    from paper_2303_05098_b200 import dist as D
    from paper_2303_05098_b200 import synth_dev
    try:
        forest = P.DeviceForest(ff)
        specs = [synth_dev.corpus_spec(i) for i in held_out_ids(count)]
        mine = D.lpt_shard([synth_dev.nnz_estimate(s) for s in specs], world, rank)
        t0 = time.perf_counter()
        rows = [profile_one(P, specs[i], forest, stream) for i in mine]
        torch.cuda.empty_cache()
        elapsed = time.perf_counter() - t0
        if world > 1:
            import torch.distributed as dist
            g = [None] * world
            dist.all_gather_object(g, (rows, elapsed))
            rows = [r for part in g for r in part[0]]
            elapsed = max(part[1] for part in g)
        return summarise_config4(sorted(rows, key=lambda r: r["id"]), elapsed, world)
    except Exception as e:
        return {"error": str(e)[:300]}


# -------------------------------------------------------------- config 5

def config5_single(P, stream, peak, iters=10):
    """27-point stencil 512^3 (DIA, 29 GB of diagonals) iterated on one GPU:
    x <- A x on two device windows, CUDA events on the stream."""
    import torch
    try:
        g = G5
        n = g ** 3
        m = P.DeviceMatrix.stencil27(g, seed=5)
        xa = torch.ones(n, dtype=torch.float64, device="cuda")
        xb = torch.empty_like(xa)
        torch.cuda.synchronize()
        for _ in range(2):
            m.spmv_device(xa.data_ptr(), xb.data_ptr(), stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for k in range(iters):
            src, dst = (xa, xb) if k % 2 == 0 else (xb, xa)
            m.spmv_device(src.data_ptr(), dst.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) * 1e-3 / iters
        nbytes = m.spmv_bytes
        # the N>1 lines' checksum protocol: x0 reloaded, CHECK_ITERS multiplies
        from paper_2303_05098_b200 import dist as D
        xa.copy_(config5_x0(0, n))
        for k in range(CHECK_ITERS):
            src, dst = (xa, xb) if k % 2 == 0 else (xb, xa)
            m.spmv_device(src.data_ptr(), dst.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        out = xa if CHECK_ITERS % 2 == 0 else xb
        csum = D.owned_checksum(out, D.partition(n, g * g + g + 1, 0, 1))
        del m, xa, xb
        torch.cuda.empty_cache()
        return {"config": config5_config(1), "iters": iters, "ms_per_iter": round(sec * 1e3, 4),
                "value": round(nbytes / sec / 1e9, 1), "unit": "GB/s", "frac": round(nbytes / sec / 1e9 / peak, 4),
                "algorithmic_bytes": nbytes, "checksum": csum,
                "checksum_protocol": CHECKSUM_PROTOCOL}
    except Exception as e:
        return {"error": str(e)[:300]}


CHECK_ITERS = 4
CHECKSUM_PROTOCOL = (f"x0[i] = 1 + (i % 7) / 8, {CHECK_ITERS} iterations of x <- A x, "
                     "sum_i (2i+1) * bits(x_i) mod 2^64 (dist.owned_checksum): identical at every N")


def config5_x0(lo, hi):
    import torch
    return 1.0 + (torch.arange(lo, hi, dtype=torch.int64, device="cuda") % 7).double() / 8.0


def run_partitioned(args, world, rank, dev):
    """N > 1: config 5 row-partitioned over the ranks (strong scaling), halo
    rows pushed into the neighbours' windows by the multiply (so_dist_*); the
    iterate's checksum is bitwise independent of N."""
    import torch
    import torch.distributed as dist
    import paper_2303_05098_b200 as P
    from paper_2303_05098_b200 import dist as D
    peak, peak_kind = peaks()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    g = G5
    n = g ** 3
    h = g * g + g + 1
    s = D.partition(n, h, rank, world)
    m = P.DeviceMatrix.stencil27(g, s.r0, s.r1, s.w0, s.w1, seed=5)
    nbytes_local = m.spmv_bytes
    it = D.make_iterator(s, m, dist, args.exchange, stream)
    it.load_x(config5_x0)
    torch.cuda.synchronize()
    dist.barrier()
    it.run(max(args.warmup, 3))
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(dev)
    clocks.start()
    from paper_2303_05098_b200 import _capi
    n0 = _capi.lib().so_kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    it.run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = _capi.lib().so_kernel_launches() - n0
    clk = clocks.stop()
    sec = e0.elapsed_time(e1) * 1e-3 / args.steps
    t = torch.tensor([sec, float(nbytes_local), float(it.timeouts())], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    tmax, tsum = t.clone(), t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    sec, nbytes = float(tmax[0]), float(tsum[1])
    # e2e: every step each rank uploads its owned rows of x from pinned host
    # memory into the iterate, runs one iteration (halos over NVLink as in the
    # device-timed loop) and reads its owned rows of the result back
    nloc = s.nloc
    xh = torch.ones(nloc, dtype=torch.float64).pin_memory()
    yh = torch.empty(nloc, dtype=torch.float64).pin_memory()

    def e2e_step():
        it.owned().copy_(xh, non_blocking=True)
        it.run(1)
        yh.copy_(it.owned(), non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e3.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e2.elapsed_time(e3) * 1e-3 / args.steps], dtype=torch.float64,
                      device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    sec_e2e = float(te[0])
    del xh, yh
    # checksum protocol shared with config5_n1 (N = 1): x0 reloaded on every
    # rank while all GPUs are idle, CHECK_ITERS iterations, then the checksum
    dist.barrier()
    it.load_x(config5_x0)
    torch.cuda.synchronize()
    dist.barrier()
    it.run(CHECK_ITERS)
    torch.cuda.synchronize()
    csum = it.checksum()
    dist.barrier()
    it.close()
    del m
    torch.cuda.empty_cache()
    cfg4 = None if args.no_config4 else config4_slice(P, stream, args.config4_count, forest_ff(), world, rank)
    if rank == 0:
        value = nbytes / sec / 1e9
        line = {"metric": "spmv_gbs", "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config5_config(world),
                "roofline": {"bound": "hbm", "achieved": round(value / world, 1), "peak": peak, "unit": "GB/s",
                             "frac": round(value / world / peak, 4), "traffic": None,
                             "algorithmic_bytes": nbytes, "kernel": "dia_kernel (+ dia_push_kernel halo rows)",
                             "peak_kind": peak_kind, "per": "GPU"},
                "exchange": it.exchange, "exchange_fallback": it.fallback, "halo_wait_timeouts": int(tsum[2]),
                "checksum": csum, "checksum_protocol": CHECKSUM_PROTOCOL, "gpu_launches": launches, "clocks": clk,
                "e2e": {"value": round(nbytes / sec_e2e / 1e9, 2), "unit": "GB/s", "ms": round(sec_e2e * 1e3, 4),
                        "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                        "call": "per step and rank: owned rows of x H2D from pinned host memory, one so_dist "
                                "iteration (NVLink halos), owned rows of the result D2H"},
                "config4_shard": cfg4}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
