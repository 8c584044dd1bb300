#!/usr/bin/env python3
"""Train with the REFERENCE's own trainer on B200 labels: the reference's
cmd_train (pipeline.cpp:190-252, compiled in place by oracle/Makefile refpipe)
reads the profile.csv / features.csv that scripts/config4.py --ref-csv wrote
in the reference's wire formats, joins them (build_training_csv: fastest
feasible format), grid-searches with k-fold CV and writes a
sparse-oracle-model v1 file that the B200 device forest loads.  Offline
tooling (test infrastructure on the reference side), not the hot path.

    python scripts/train_reference.py gpurun_out/c4ref --out /tmp/ref_forest.txt
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dir")
    ap.add_argument("--out", required=True)
    ap.add_argument("--seed", type=int, default=2303)
    ap.add_argument("--folds", type=int, default=5)
    a = ap.parse_args()
    rep = oracle.ref_cmd_train(os.path.join(a.dir, "features.csv"), os.path.join(a.dir, "profile.csv"), a.out,
                               seed=a.seed, folds=a.folds)
    print(json.dumps(rep))


if __name__ == "__main__":
    main()
