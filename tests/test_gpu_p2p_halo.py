"""Fused peer-memory halo exchange (config 5, dist.PeerWindows): the multiply
of the boundary rows stores them straight into the neighbour's window
(so_spmv_rows_push over CUDA IPC) and publishes a release/acquire flag; no
collective on the data path.  Two and three ranks run as separate processes
sharing the one GPU of the box (CUDA IPC between processes on one device),
bootstrapped over gloo on 127.0.0.1; the P-rank iterate must be bitwise equal
to the 1-rank iterate (the row partition does not change any row's order)."""
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


def _rank_main(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import paper_2303_05098_b200 as P
    from paper_2303_05098_b200 import dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    P.set_device(0)
    n, h = G ** 3, G * G + G + 1
    s = D.partition(n, h, rank, world)
    m = P.DeviceMatrix.stencil27(G, s.r0, s.r1, s.w0, s.w1, seed=SEED)
    pw = D.PeerWindows(s, dist.all_gather_object)
    stream = torch.cuda.Stream()
    pw.tensor(0).copy_(torch.from_numpy(_x0(s.w0, s.w1)))
    torch.cuda.synchronize()
    dist.barrier()
    k = pw.iterate(m, ITERS, stream.cuda_stream)
    stream.synchronize()
    assert pw.timeouts() == 0
    own = pw.tensor(k)[s.own_lo:s.own_hi].cpu().numpy()
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), own)
    dist.barrier()  # peers keep their mappings until everyone is done
    pw.close()
    dist.destroy_process_group()


def _one_rank_reference():
    import torch

    import paper_2303_05098_b200 as P

    n = G ** 3
    m = P.DeviceMatrix.stencil27(G, seed=SEED)
    xa = torch.tensor(_x0(0, n), device="cuda")
    xb = torch.empty_like(xa)
    torch.cuda.synchronize()  # the library's stream does not wait for torch's
    for _ in range(ITERS):
        m.spmv_device(xa.data_ptr(), xb.data_ptr())
        xa, xb = xb, xa
    torch.cuda.synchronize()
    return xa.cpu().numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_halo_iteration_bitwise(world, tmp_path):
    import torch.multiprocessing as mp

    want = _one_rank_reference()
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0, f"rank process failed ({p.exitcode})"
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])
    assert got.shape == want.shape
    assert np.array_equal(got, want)
