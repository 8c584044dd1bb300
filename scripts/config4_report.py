#!/usr/bin/env python3
"""Summarise a config-4 tuned run (scripts/config4.py --model): tuner accuracy
vs the measured-optimal format, tuning cost in CSR-SpMV equivalents
((T_FE+T_PRED)/t_CSR, pipeline.cpp:300-302), and the Eq. 2 speedup
T_CSR/(T_FE+T_PRED+T_OPT) with 1000 repetitions (pipeline.cpp:298-299)."""
import csv
import json
import sys

import numpy as np

FMT = ["COO", "CSR", "DIA", "ELL", "HYB", "HDC"]


def main(path, reps=1000):
    rows = list(csv.DictReader(open(path)))
    lab = np.array([int(r["label"]) for r in rows])
    ch = np.array([int(r["chosen"]) for r in rows])
    t = np.array([[float(r["t_" + f]) for f in FMT] for r in rows])
    tfe = np.array([float(r["t_fe"]) for r in rows])
    tpr = np.array([float(r["t_pred"]) for r in rows])
    idx = np.arange(len(rows))
    t_opt, t_ch, t_csr = t.min(1), t[idx, ch], t[:, 1]
    cost = (tfe + tpr) / t_csr
    speedup = (reps * t_csr) / (tfe + tpr + reps * t_ch)
    recalls = [float((ch[lab == c] == c).mean()) for c in range(6) if (lab == c).any()]
    q = np.quantile(cost, [0, 0.25, 0.5, 0.75, 1])
    out = {
        "matrices": len(rows),
        "accuracy": float((ch == lab).mean()),
        "balanced_accuracy": float(np.mean(recalls)),
        "within_5pct_of_optimal": float((t_ch <= 1.05 * t_opt).mean()),
        "mean_slowdown_vs_optimal": float((t_ch / t_opt).mean()),
        "tuning_cost_csr_spmv_equiv": {"mean": float(cost.mean()), "min": q[0], "q1": q[1], "median": q[2],
                                       "q3": q[3], "max": q[4]},
        "eq2_speedup_1000reps": {"mean": float(speedup.mean()), "geomean": float(np.exp(np.log(speedup).mean())),
                                 "max": float(speedup.max()), "frac_gt_1": float((speedup > 1).mean())},
        "spmv_only_speedup_vs_csr_geomean": float(np.exp(np.log(t_csr / t_ch).mean())),
        "oracle_speedup_vs_csr_geomean": float(np.exp(np.log(t_csr / t_opt).mean())),
        "t_fe_ms_median": float(np.median(tfe) * 1e3), "t_pred_ms_median": float(np.median(tpr) * 1e3),
    }
    if rows and "t_wall" in rows[0] and rows[0]["t_wall"]:  # host wall clock of the tune_ml call
        tw = np.array([float(r["t_wall"]) for r in rows])
        cw = tw / t_csr
        qw = np.quantile(cw, [0, 0.25, 0.5, 0.75, 1])
        out["tuning_cost_csr_spmv_equiv_wall"] = {"mean": float(cw.mean()), "min": qw[0], "q1": qw[1],
                                                  "median": qw[2], "q3": qw[3], "max": qw[4],
                                                  "frac_below_10": float((cw < 10).mean())}
        out["tuning_cost_csr_spmv_equiv"]["frac_below_10"] = float((cost < 10).mean())
    print(json.dumps(out, indent=1))
    return out


if __name__ == "__main__":
    main(sys.argv[1])
