#!/usr/bin/env python3
"""Per-matrix tuning cost on the held-out config-4 slice (bench.py's
profile_one): device T_FE + T_PRED and host wall clock, in CSR-SpMV
equivalents; the worst matrices first.  `--ids a,b` re-runs only those (e.g.
under an ncu launch list)."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (puts the repo root first on sys.path)

if os.environ.get("AB_ROOT"):  # an A/B variant package (scripts/ab_build.sh) ahead of the repo's
    sys.path.insert(0, os.environ["AB_ROOT"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ids", default="")
    ap.add_argument("--count", type=int, default=100)
    a = ap.parse_args()
    import torch
    import paper_2303_05098_b200 as P
    from paper_2303_05098_b200 import synth_dev
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    forest = P.DeviceForest(bench.forest_ff())
    ids = [int(i) for i in a.ids.split(",")] if a.ids else bench.held_out_ids(a.count)
    rows = []
    for i in ids:
        r = bench.profile_one(P, synth_dev.corpus_spec(i), forest, stream)
        tc = r["t"][1] / r["reps"]
        r["cost"] = (r["t_fe"] + r["t_pred"]) / tc
        r["cost_w"] = r["t_wall"] / tc
        r["t_csr"] = tc
        rows.append(r)
    rows.sort(key=lambda r: -r["cost_w"])
    for r in rows[:25]:
        print(json.dumps({k: (round(v, 7) if isinstance(v, float) else v) for k, v in r.items()
                          if k in ("id", "family", "n", "nnz", "t_csr", "t_fe", "t_pred", "t_wall", "cost", "cost_w",
                                   "label", "chosen")}))
    c = np.array([r["cost_w"] for r in rows])
    print("wall cost mean %.3f median %.3f max %.3f" % (c.mean(), np.median(c), c.max()))


if __name__ == "__main__":
    main()
