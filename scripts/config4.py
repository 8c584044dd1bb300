#!/usr/bin/env python3
"""Config 4: a batch of synthetic matrices (stencil / banded / uniform-random /
power-law, 10K-5M rows) -> device features + measured-optimal format on the
B200 (run-first profiling, tuners.cpp:47-90 semantics: argmin total time,
ties to the lowest id) -> CSV, and optionally the device ML tuner's choice
with its T_FE / T_PRED.

Sharded over ranks when launched with torchrun: greedy LPT by nnz estimate,
no data-path collective; rows are gathered on rank 0 at the end.

    python scripts/config4.py --count 400 --reps 20 --out profiles/config4_r1.csv
    python scripts/config4.py ... --model paper_2303_05098_b200/models/b200_forest.txt
"""
from __future__ import annotations

import argparse
import csv
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth_dev  # noqa: E402

FMT = P.FORMAT_NAMES


def lpt_shard(specs, world, rank):
    from paper_2303_05098_b200 import dist as D
    idx = D.lpt_shard([synth_dev.nnz_estimate(s) for s in specs], world, rank)
    return sorted((specs[i] for i in idx), key=lambda s: s["id"])


def time_format(m, x, y, reps, stream):
    """reps back-to-back multiplies after one warm-up, each timed with a CUDA
    event pair on the launching stream (time_spmv semantics)."""
    m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    for r in range(reps):
        m.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
        ev[r + 1].record(stream)
    ev[-1].synchronize()
    return [ev[r].elapsed_time(ev[r + 1]) * 1e-3 for r in range(reps)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=2000)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="profiles/config4.csv")
    ap.add_argument("--model", default=None)
    ap.add_argument("--nmax", type=int, default=5_000_000)
    ap.add_argument("--only", default=None, help="JSON with test_ids: restrict to the held-out matrices")
    ap.add_argument("--ref-csv", default=None,
                    help="directory: also write profile.csv / features.csv in the reference's wire "
                         "formats (ingest.cpp:419-470) for the reference trainer (cmd_train)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    P.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    forest = None
    if a.model:
        from paper_2303_05098_b200 import forest as F
        forest = P.DeviceForest(F.load_model(a.model))

    specs = [synth_dev.corpus_spec(i, nmax=a.nmax) for i in range(a.start, a.start + a.count)]
    if a.only:
        import json
        keep = set(json.load(open(a.only))["test_ids"])
        specs = [s for s in specs if s["id"] in keep]
    mine = lpt_shard(specs, world, rank)
    rows = []
    t_start = time.perf_counter()
    for s in mine:
        csr = synth_dev.build(s)
        base = csr.to_device_matrix()
        del csr
        fv = base.extract_features(0.2)
        x = torch.ones(fv.ncols, dtype=torch.float64, device="cuda")
        y = torch.empty(fv.nrows, dtype=torch.float64, device="cuda")
        tot, mats = {}, {}
        for f in range(6):
            try:
                mats[f] = base.convert(f)
            except P.PaddingOverflow:
                tot[f] = float("inf")
                continue
            tot[f] = float(np.sum(time_format(mats[f], x, y, a.reps, stream)))
        twins = P.kernel_twins(mats)
        del mats
        label = min(range(6), key=lambda f: (tot[f], f))
        # twins run the same kernel on the same arrays: one time for both (the
        # faster measurement), so every argmin -- ours and the reference
        # trainer's build_training_csv -- breaks the tie toward the lowest id
        tot_c = dict(tot)
        for f, t in twins.items():
            tot_c[f] = tot_c[t] = min(tot[f], tot[t])
        row_ref = (f"c4_{s['id']:04d}", [(f, a.reps, tot_c[f], tot[f] != float("inf")) for f in range(6)])
        row = {"id": s["id"], "family": s["family"], "n": fv.nrows, "nnz": fv.nnz}
        row.update({f"f{k}": v for k, v in enumerate(fv.to_row())})
        row.update({f"t_{FMT[f]}": tot[f] / a.reps for f in range(6)})
        row["label"] = label
        row["label_collapsed"] = min(range(6), key=lambda f: (tot_c[f], f))
        row["twins"] = ";".join(f"{f}-{t}" for f, t in sorted(twins.items()) if f < t)
        if forest is not None:
            P.tune_ml(base, forest)  # warm-up (forest already resident)
            outs = [P.tune_ml(base, forest) for _ in range(3)]
            o = outs[-1]
            row["chosen"] = int(o.chosen)
            row["t_fe"] = float(np.median([q.feature_time_seconds for q in outs]))
            row["t_pred"] = float(np.median([q.predict_time_seconds for q in outs]))
            row["t_wall"] = float(np.median([q.wall_time_seconds for q in outs]))
        row["_ref"] = row_ref
        rows.append(row)
        del base
    elapsed = time.perf_counter() - t_start
    if world > 1:
        import torch.distributed as dist
        gathered = [None] * world
        dist.all_gather_object(gathered, (rows, elapsed))
        rows = [r for g in gathered for r in g[0]]
        elapsed = max(g[1] for g in gathered)
    if rank == 0:
        rows.sort(key=lambda r: r["id"])
        if a.ref_csv:
            from paper_2303_05098_b200 import wire
            os.makedirs(a.ref_csv, exist_ok=True)
            wire.write_profile_csv(os.path.join(a.ref_csv, "profile.csv"),
                                   [(mid, f, reps, t, ok) for r in rows for mid, recs in [r["_ref"]]
                                    for f, reps, t, ok in recs])
            wire.write_feature_csv(os.path.join(a.ref_csv, "features.csv"),
                                   [(r["_ref"][0], [r[f"f{k}"] for k in range(10)]) for r in rows])
        for r in rows:
            r.pop("_ref", None)
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
            w.writeheader()
            w.writerows(rows)
        labels = np.bincount([r["label"] for r in rows], minlength=6)
        print(f"rank0: {len(rows)} matrices on {world} GPU(s) in {elapsed:.1f}s "
              f"({len(rows) / elapsed:.2f} matrices/s); measured-optimal distribution "
              + ", ".join(f"{FMT[f]}={labels[f]}" for f in range(6)), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
