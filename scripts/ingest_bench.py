#!/usr/bin/env python3
"""SURVEY §8 f1 on the B200 host: Matrix Market ingest and triplet
canonicalization, the reference (oracle/_ref: its read_matrix_market and
CooMatrix::from_triplets compiled in place) vs this library
(so_read_matrix_market: host-parallel parse + device canonicalization;
so_coo_from_triplets: device radix sort with in-order duplicate sums).

* read: a Matrix Market file of the config-1 Laplacian and of an R-MAT
  2^21 (written once with the reference's writer), wall time per read,
  results checked equal;
* from_triplets: the config-3 R-MAT entries (65 M) in a random order with
  duplicates, wall time, canonical arrays checked equal.

Measurement script (test infrastructure may be imported here: it times the
reference, it is not the product path).

    python scripts/ingest_bench.py > profiles/rNN_ingest.json
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle as O  # noqa: E402
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402


def timed(fn, reps=1):
    best = None
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return out, best


def main():
    res = {"host_threads": os.cpu_count(), "read_matrix_market": {}, "from_triplets": {}}
    with tempfile.TemporaryDirectory() as d:
        for name, csr in (("laplacian 1000^2 (config 1)", synth.laplacian_2d(1000, seed=1)),
                          ("rmat 2^21 d16", synth.rmat(21, 16, seed=7))):
            coo = O.coo_dict(csr.nrows, csr.ncols, csr.coo_rows(), csr.col, csr.val)
            path = os.path.join(d, "m.mtx")
            O.ref_write_matrix_market(path, coo)
            size = os.path.getsize(path)
            (st, ref), t_ref = timed(lambda: O.ref_read_matrix_market(path))
            assert st == "ok", st
            ours, t_ours = timed(lambda: P.DeviceMatrix.read_matrix_market(path), reps=3)
            got = ours.download()
            same = all(np.array_equal(got[k], ref[k]) for k in ("row", "col", "val"))
            res["read_matrix_market"][name] = {"file_mb": round(size / 1e6, 1), "nnz": int(coo["val"].size),
                                               "reference_s": round(t_ref, 3), "b200_s": round(t_ours, 4),
                                               "speedup": round(t_ref / t_ours, 1), "identical": bool(same)}
            # write_matrix_market: the reference's writer vs ours (same bytes)
            p2 = os.path.join(d, "w.mtx")
            _, tw_ref = timed(lambda: O.ref_write_matrix_market(path, coo))
            _, tw_ours = timed(lambda: ours.write_matrix_market(p2), reps=3)
            with open(path, "rb") as fa, open(p2, "rb") as fb:
                same_w = fa.read() == fb.read()
            res.setdefault("write_matrix_market", {})[name] = {
                "reference_s": round(tw_ref, 3), "b200_s": round(tw_ours, 4), "speedup": round(tw_ref / tw_ours, 1),
                "byte_identical": bool(same_w)}
            print(name, res["read_matrix_market"][name], file=sys.stderr, flush=True)
    csr = synth.rmat(22, 16, seed=42)
    r, c, v = csr.coo_rows(), csr.col.astype(np.int64), csr.val
    rng = np.random.default_rng(3)
    # one duplicate for 3 % of the entries (two terms per key: their sum is
    # the same in any order, so both sides must agree bit for bit)
    dup = rng.choice(r.size, r.size // 32, replace=False)
    r = np.concatenate([r, r[dup]])
    c = np.concatenate([c, c[dup]])
    v = np.concatenate([v, 0.5 * v[dup]])
    perm = rng.permutation(r.size)
    r, c, v = r[perm], c[perm], v[perm]
    ref_m, t_ref = timed(lambda: O.RefMatrix.from_triplets(csr.nrows, csr.ncols, r, c, v))
    ours, t_ours = timed(lambda: P.DeviceMatrix.from_triplets(csr.nrows, csr.ncols, r, c, v), reps=3)
    e, g = ref_m.export(), ours.download()
    same = all(np.array_equal(g[k], e[k]) for k in ("row", "col", "val"))
    res["from_triplets"]["rmat 2^22 d16 (config 3), shuffled, +3% duplicates"] = {
        "triplets": int(r.size), "reference_s": round(t_ref, 3), "b200_s": round(t_ours, 4),
        "speedup": round(t_ref / t_ours, 1), "identical": bool(same)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
