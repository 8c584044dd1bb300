#!/usr/bin/env python3
"""compute-sanitizer driver: every kernel of the library on small inputs, no
torch (so the tool sees only this library's kernels).

    compute-sanitizer --tool memcheck  python scripts/sanitize_driver.py
    compute-sanitizer --tool racecheck python scripts/sanitize_driver.py
    compute-sanitizer --tool synccheck python scripts/sanitize_driver.py
    compute-sanitizer --tool memcheck --target-processes all python scripts/sanitize_driver.py dist2

Covers: uploads / downloads, every conversion pair, the six SpMV kernels
(CSR warp groups plain / padded / cooperative, long-row pieces + fix-up, COO
chunk fix-up incl. queued long runs and the empty-row-gap path, DIA with <= 5
and > 5 diagonals, ELL, HYB, HDC both parts), the pageable staging path
(zero-copy DIA row blocks and the copy-engine path), pinned host buffers (the
follow-the-copy DIA kernel), features on every format
(both spread-walk variants, entry and lockstep sweeps, big-row pieces),
predict (flat and blocked), the tune graph, device from_triplets, Matrix
Market I/O, the halo push / flag wait kernels and so_dist (1 rank; 2 ranks in
two processes with `dist2`).
"""
import ctypes as C
import os
import sys
import tempfile

# the pinned-buffer case exercises the follow-the-copy kernel even under the
# sanitizer (which may serialise it against the copy: the call then times out
# and falls back -- slower, still correct)
os.environ.setdefault("SOB_FOLLOW_UNDER_TOOLS", "1")

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import _capi as A  # noqa: E402
from paper_2303_05098_b200 import dist as D  # noqa: E402
from paper_2303_05098_b200 import synth  # noqa: E402


_pinned_keep = []


def pinned(n):
    """n doubles of pinned, mapped host memory (cudaHostAlloc through the
    CUDA runtime's shared library; no torch), or None when unavailable."""
    for name in ("libcudart.so", "/usr/local/cuda/lib64/libcudart.so", "libcudart.so.12"):
        try:
            rt = C.CDLL(name)
            break
        except OSError:
            rt = None
    if rt is None:
        return None
    p = C.c_void_p()
    if rt.cudaHostAlloc(C.byref(p), C.c_size_t(8 * n), C.c_uint(2)) != 0:  # cudaHostAllocMapped
        return None
    _pinned_keep.append((rt, p))
    return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(n,))


def csr_from(n, m, rows, cols, rng):
    rows, cols = np.asarray(rows, np.int64), np.asarray(cols, np.int64)
    key = np.unique(rows * m + cols)
    r, c = key // m, key % m
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    np.cumsum(rp, out=rp)
    return synth.HostCSR(n, m, rp, c, rng.uniform(0.5, 2.0, c.size) * rng.choice([-1.0, 1.0], c.size))


def shapes(rng):
    n = 2000
    out = {"band13": synth.banded(n, 13, seed=1), "lap": synth.laplacian_2d(30, seed=2),
           "stencil": synth.stencil_3d(10, 27, seed=3), "rmat": synth.rmat(11, 8, seed=4),
           "even16": synth.hyb_skewed(n, 16, 16, 100, seed=5), "hyb": synth.hyb_skewed(n, 6, 90, 17, seed=6)}
    # one dense row far past the warp-group cap (long-row pieces) + a dense column
    r = np.concatenate([np.arange(n), np.full(n, 5), np.arange(n)])
    c = np.concatenate([np.arange(n), np.arange(n), np.full(n, 7)])
    out["arrow"] = csr_from(n, n, r, c, rng)
    # rows spanning > 64 COO chunks (queued long runs) and a > 4096-row empty gap
    big = 70 * 256 + 3
    r = np.concatenate([np.zeros(big, np.int64), np.full(10, 9000)])
    c = np.concatenate([np.arange(big) % 20000, np.arange(10)])
    out["longrun_gap"] = csr_from(10000, 20000, r, c, rng)
    return out


def exercise(name, csr, forest, x_rng, pairs):
    x = x_rng.uniform(-1, 1, csr.ncols)
    base = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    for f in range(6):
        try:
            m = base.convert(f)
        except P.PaddingOverflow:
            continue
        m.download()
        m.spmv(x)
        m.extract_features(0.2)
        if f == 1:
            m.time_spmv(x, 1)
            P.tune_ml(m, forest)
            P.tune_ml(m, forest)  # graph replay
        if pairs:  # every conversion pair (X -> CSR -> Y) once
            for g in range(6):
                try:
                    m.convert(g).to_coo()
                except P.PaddingOverflow:
                    pass
    print("ok", name, flush=True)


def push_and_wait():
    lib = A.lib()
    csr = synth.banded(4096, 3, seed=9)
    m = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val).convert(P.DIA)
    bufs = []
    for nbytes in (8 * 4096, 8 * 4096, 8 * 4096, 64):
        p, h = C.c_void_p(), C.create_string_buffer(64)
        assert lib.so_ipc_alloc(nbytes, C.byref(p), h) == 0
        bufs.append(p.value)
    x, y, remote, flags = bufs
    st = lib.so_spmv_rows_push(m._h, C.c_void_p(x), C.c_void_p(y), 0, 64, C.c_void_p(remote),
                               C.c_void_p(flags + 32), C.c_void_p(flags), 1, None)
    assert st == 0, lib.so_last_error()
    assert lib.so_wait_flag(C.c_void_p(flags), 1, None) == 0
    assert lib.so_device_sync() == 0
    for p in bufs:
        lib.so_ipc_free(C.c_void_p(p))
    # so_dist with one rank: HALO (interior only) and ALLGATHER (no peers)
    g = 10
    n, h = g ** 3, g * g + g + 1
    st27 = P.DeviceMatrix.stencil27(g, seed=3)
    it = D.DistIteration(st27, D.HALO, 0, 1, [0, n], h, lambda out, obj: out.__setitem__(0, obj))
    it.iterate(3)
    it.close()
    rm = synth.rmat(10, 6, seed=3)
    cm = P.DeviceMatrix.csr(rm.nrows, rm.ncols, rm.row_ptr, rm.col, rm.val)
    it = D.DistIteration(cm, D.ALLGATHER, 0, 1, [0, rm.nrows], 0, lambda out, obj: out.__setitem__(0, obj))
    it.iterate(3)
    it.close()
    assert lib.so_device_sync() == 0
    print("ok push/wait/dist1", flush=True)


def _dist_rank(rank, conn, kind):
    P.set_device(0)
    if kind == "halo":
        g = 12
        n, h = g ** 3, g * g + g + 1
        s = D.partition(n, h, rank, 2)
        m = P.DeviceMatrix.stencil27(g, s.r0, s.r1, s.w0, s.w1, seed=3)
        st, halo, k = D.row_starts(n, 2), h, D.HALO
    else:
        rm = synth.rmat(10, 6, seed=3)
        st = D.row_starts(rm.nrows, 2)
        a, b = st[rank], st[rank + 1]
        m = P.DeviceMatrix.csr(b - a, rm.ncols, rm.row_ptr[a:b + 1] - rm.row_ptr[a],
                               rm.col[rm.row_ptr[a]:rm.row_ptr[b]], rm.val[rm.row_ptr[a]:rm.row_ptr[b]])
        halo, k = 0, D.ALLGATHER

    def all_gather(out, obj):
        conn.send(obj)
        other = conn.recv()
        out[rank], out[1 - rank] = obj, other

    it = D.DistIteration(m, k, rank, 2, st, halo, all_gather)
    conn.send("ready")
    conn.recv()
    it.iterate(4)
    assert A.lib().so_device_sync() == 0
    assert it.timeouts() == 0
    conn.send("done")
    conn.recv()
    it.close()


def dist2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    for kind in ("halo", "allgather"):
        a, b = ctx.Pipe()
        ps = [ctx.Process(target=_dist_rank, args=(0, a, kind)), ctx.Process(target=_dist_rank, args=(1, b, kind))]
        for p in ps:
            p.start()
        for p in ps:
            p.join(timeout=600)
            assert p.exitcode == 0, (kind, p.exitcode)
        print("ok dist2", kind, flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "dist2":
        return dist2()
    quick = "--quick" in sys.argv  # the pytest gate: every kernel, fewer shapes
    rng = np.random.default_rng(0)
    from paper_2303_05098_b200.models import default_forest
    ff = default_forest()
    forest = P.DeviceForest(ff)
    forest.predict_rows(rng.uniform(0, 1e6, (64, 10)))
    forest.predict_rows_latency(rng.uniform(0, 1e6, (64, 10)))
    for name, csr in shapes(rng).items():
        if quick and name in ("band13", "stencil", "even16"):
            continue
        exercise(name, csr, forest, rng, pairs=name == "hyb" or (not quick and name == "stencil"))
    # pageable staging: zero-copy DIA row blocks and the copy-engine path
    big = synth.banded(140_000, 4, seed=7)
    bm = P.DeviceMatrix.csr(big.nrows, big.ncols, big.row_ptr, big.col, big.val)
    xb = rng.uniform(-1, 1, big.ncols)
    for f in (P.DIA, P.CSR, P.COO):
        bm.convert(f).spmv(xb)
    # pinned host buffers: the follow-the-copy kernel (and, with
    # SOB_NO_FOLLOW=1, the zero-copy kernel) on a narrow DIA window
    # (>= 2^19 rows: smaller calls take the one-shot path)
    band = synth.banded(600_000, 4, seed=9)
    bcsr = P.DeviceMatrix.csr(band.nrows, band.ncols, band.row_ptr, band.col, band.val)
    hx, hy = pinned(band.ncols), pinned(band.nrows)
    if hx is not None and hy is not None:
        hx[:] = rng.uniform(-1, 1, band.ncols)
        for fmt in (P.DIA, P.CSR, P.ELL, P.COO):  # DIA / CSR / ELL follow kernels, the pinned one-shot path
            dm = bcsr.convert(fmt)
            for _ in range(2):
                dm.spmv_into(hx, hy)
                assert np.array_equal(hy, dm.spmv(np.array(hx))), "pinned spmv differs from the one-shot path"
    # large enough for the global-memory spread walk and the lockstep sweep
    big2 = synth.uniform_random(60_000, 5, seed=8)
    P.DeviceMatrix.csr(big2.nrows, big2.ncols, big2.row_ptr, big2.col, big2.val).extract_features(0.2)
    # device from_triplets (radix sort + duplicate sums) and Matrix Market I/O
    r = rng.integers(0, 500, 4000)
    c = rng.integers(0, 700, 4000)
    coo = P.DeviceMatrix.from_triplets(500, 700, r, c, rng.uniform(-1, 1, 4000))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "m.mtx")
        coo.write_matrix_market(path)
        P.DeviceMatrix.read_matrix_market(path).convert(P.CSR)
    push_and_wait()
    print("sanitize driver done", flush=True)


if __name__ == "__main__":
    main()
