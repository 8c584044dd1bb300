#!/usr/bin/env python3
"""Train the device tuner's forest on B200 profiling labels (config 4).

Seeded 80/20 split (cmd_train semantics, pipeline.cpp:203-212), CART forest
(paper_2303_05098_b200/forest.py), held-out accuracy / balanced accuracy
against the measured-optimal format, model written in the reference text
format.  Offline tooling, not the hot path.

    python scripts/train_forest.py profiles/config4_profile_2000.csv \
        --out paper_2303_05098_b200/models/b200_forest.txt
"""
import argparse
import csv
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05098_b200 import forest as F  # noqa: E402


def load(path):
    with open(path) as f:
        rows = list(csv.DictReader(f))
    X = np.array([[float(r[f"f{k}"]) for k in range(10)] for r in rows])
    key = "label_collapsed" if rows and "label_collapsed" in rows[0] else "label"
    y = np.array([int(r[key]) for r in rows])
    return rows, X, y


def split(n, seed):
    rng = np.random.default_rng(seed)
    idx = rng.permutation(n)
    cut = int(round(0.8 * n))
    return np.sort(idx[:cut]), np.sort(idx[cut:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out", default="paper_2303_05098_b200/models/b200_forest.txt")
    ap.add_argument("--trees", type=int, default=50)
    ap.add_argument("--depth", type=int, default=16)
    ap.add_argument("--seed", type=int, default=2303)
    ap.add_argument("--split-out", default=None, help="write held-out ids as JSON")
    a = ap.parse_args()
    rows, X, y = load(a.csv)
    tr, te = split(len(y), a.seed)
    ff = F.train_forest(X[tr], y[tr], n_estimators=a.trees, max_depth=a.depth, seed=a.seed)
    pred = F.predict_rows_host(ff, X[te])
    ev = F.evaluate(y[te], pred)
    tree = F.flatten([F.train_tree(X[tr], y[tr], max_depth=a.depth)], kind=0)
    ev_tree = F.evaluate(y[te], F.predict_rows_host(tree, X[te]))
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    meta = [("backend", "b200-sm_100a"), ("labels", os.path.basename(a.csv)),
            ("n_train", str(len(tr))), ("n_estimators", str(a.trees)), ("max_depth", str(a.depth)),
            ("seed", str(a.seed))]
    F.save_model(ff, a.out, meta)
    F.save_model(tree, a.out.replace(".txt", "_tree.txt"), meta)
    summary = {"n_train": int(len(tr)), "n_test": int(len(te)), "forest": ev, "tree": ev_tree,
               "label_distribution": np.bincount(y, minlength=6).tolist(), "model": a.out,
               "test_ids": [int(rows[i]["id"]) for i in te]}
    if a.split_out:
        with open(a.split_out, "w") as f:
            json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "test_ids"}))


if __name__ == "__main__":
    main()
