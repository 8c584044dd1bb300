"""Row-partitioned iterated SpMV through the library's so_dist_* entry points
(csrc/dist.cu, config 5 and its non-banded generalisation):

* HALO (27-point stencil, DIA): the multiply of the boundary rows stores them
  straight into the neighbour's window over peer memory and publishes a
  release/acquire flag; no collective on the data path;
* ALLGATHER (R-MAT / uniform-random rows, CSR and COO): each rank's new rows
  are stored into every peer's x by the iteration's epilogue kernel.

Two and three ranks run as separate processes sharing the one GPU of the box
(CUDA IPC between processes on one device), bootstrapped over gloo on
127.0.0.1; the P-rank iterate must be bitwise equal to the 1-rank iterate
(CSR: the row partition does not change any row's order) or within the SpMV
bar (COO: chunk boundaries move with the partition)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = 16          # 16^3 = 4096 rows, halo h = 273
ITERS = 5
SEED = 7


def _x0(lo, hi):
    return 1.0 + (np.arange(lo, hi) % 7) / 8.0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_dir, kind="halo", fmt=1):
    import torch
    import torch.distributed as dist

    import paper_2303_05098_b200 as P
    from paper_2303_05098_b200 import dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    P.set_device(0)
    stream = torch.cuda.Stream()
    if kind == "halo":
        n, h = G ** 3, G * G + G + 1
        s = D.partition(n, h, rank, world)
        m = P.DeviceMatrix.stencil27(G, s.r0, s.r1, s.w0, s.w1, seed=SEED)
        it = D.DistIteration(m, D.HALO, rank, world, D.row_starts(n, world), h, dist.all_gather_object)
        lo, hi = s.w0, s.w1
    else:
        csr = _general(kind)
        n = csr.nrows
        st = D.row_starts(n, world)
        r0, r1 = st[rank], st[rank + 1]
        rp = csr.row_ptr[r0:r1 + 1] - csr.row_ptr[r0]
        sl = slice(int(csr.row_ptr[r0]), int(csr.row_ptr[r1]))
        m = P.DeviceMatrix.csr(r1 - r0, n, rp, csr.col[sl], csr.val[sl])
        if fmt != 1:
            m = m.convert(fmt)
        it = D.DistIteration(m, D.ALLGATHER, rank, world, st, 0, dist.all_gather_object)
        lo, hi = 0, n
        s = D.Slice(n, 0, rank, world, r0, r1, 0, n)
    it.tensor(0).copy_(torch.from_numpy(_x0(lo, hi)))
    torch.cuda.synchronize()
    dist.barrier()
    it.iterate(ITERS, stream.cuda_stream)
    stream.synchronize()
    assert it.timeouts() == 0
    own = it.tensor(-1)[s.r0 - s.w0:s.r1 - s.w0].cpu().numpy()
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), own)
    dist.barrier()  # peers keep their mappings until everyone is done
    it.close()
    dist.destroy_process_group()


def _general(kind):
    from paper_2303_05098_b200 import synth
    if kind == "rmat":
        return synth.rmat(12, 6, seed=21)
    return synth.uniform_random(5000, 7, seed=22)


def _iterate_full(m, n):
    import torch
    xa = torch.tensor(_x0(0, n), device="cuda")
    xb = torch.empty_like(xa)
    torch.cuda.synchronize()  # the library's stream does not wait for torch's
    for _ in range(ITERS):
        m.spmv_device(xa.data_ptr(), xb.data_ptr())
        xa, xb = xb, xa
    torch.cuda.synchronize()
    return xa.cpu().numpy()


def _one_rank_reference():
    import paper_2303_05098_b200 as P
    return _iterate_full(P.DeviceMatrix.stencil27(G, seed=SEED), G ** 3)


def _spawn(world, tmp_path, *extra):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, str(tmp_path), *extra)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0, f"rank process failed ({p.exitcode})"
    return np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])


@pytest.mark.parametrize("world", [2, 3])
def test_fused_halo_iteration_bitwise(world, tmp_path):
    want = _one_rank_reference()
    got = _spawn(world, tmp_path)
    assert got.shape == want.shape
    assert np.array_equal(got, want)


@pytest.mark.parametrize("kind,fmt,world", [("rmat", 1, 2), ("rmat", 1, 3), ("uniform", 1, 3),
                                            ("uniform", 0, 2)])
def test_allgather_iteration(kind, fmt, world, tmp_path):
    import paper_2303_05098_b200 as P
    csr = _general(kind)
    full = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
    if fmt != 1:
        full = full.convert(fmt)
    want = _iterate_full(full, csr.nrows)
    got = _spawn(world, tmp_path, kind, fmt)
    assert got.shape == want.shape
    if fmt == 1:  # CSR rows keep their order under any row partition
        assert np.array_equal(got, want)
    else:
        assert np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) <= 1e-12
