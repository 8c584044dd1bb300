"""CPU (gloo, world_size 2 and 3): the row-partition / halo-exchange host
logic of the config-5 iteration (paper_2303_05098_b200/dist.py) reproduces
the single-rank iterate BIT-FOR-BIT.  The multiply here is a numpy restatement
of the per-row DIA order; on the GPU path the same `iterate` drives the
sm_100a row-range DIA kernel and NCCL point-to-point (scripts/config5.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_05098_b200 import dist as D

G = 6
N = G ** 3
H = G * G + G + 1
OFFS = [(k // 9 - 1) * G * G + ((k // 3) % 3 - 1) * G + (k % 3 - 1) for k in range(27)]


def value(i, d):
    z, y, x = i // (G * G), (i // G) % G, i % G
    dz, dy, dx = d // 9 - 1, (d // 3) % 3 - 1, d % 3 - 1
    if not (0 <= z + dz < G and 0 <= y + dy < G and 0 <= x + dx < G):
        return 0.0
    return 0.5 + ((i * 27 + d) * 2654435761 % 1000) / 1000.0 * (1 if (i + d) % 2 else -1)


def make_local(s):
    vals = np.array([[value(s.r0 + il, d) for il in range(s.nloc)] for d in range(27)])
    return vals, D.local_offsets(OFFS, s)


def spmv_rows_factory(s, vals, offs):
    def spmv_rows(xw, yw, lo, hi):
        for il in range(lo, hi):
            acc = 0.0
            for d in range(27):  # diagonals ascending, in-range only (spmv.cpp:45-56)
                c = il + offs[d]
                if 0 <= c < s.nwin:
                    acc = acc + vals[d, il] * xw[c]
            yw[s.own_lo + il] = acc
    return spmv_rows


def x0(i):
    return 1.0 + (i % 7) / 8.0


def run_single(iters):
    s = D.partition(N, H, 0, 1)
    vals, offs = make_local(s)
    xa = np.array([x0(s.w0 + k) for k in range(s.nwin)])
    xb = np.zeros_like(xa)
    return D.iterate(s, xa, xb, iters, spmv_rows_factory(s, vals, offs), lambda buf, plan: None)


def worker(rank, world, port, iters, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    s = D.partition(N, H, rank, world)
    vals, offs = make_local(s)
    xa = np.array([x0(s.w0 + k) for k in range(s.nwin)])
    xb = np.zeros_like(xa)

    def exchange(buf, plan):
        reqs, recvs = [], []
        for peer, (sa, sb), (ra, rb) in plan:
            reqs.append(dist.isend(torch.from_numpy(buf[sa:sb].copy()), peer))
            t = torch.empty(rb - ra, dtype=torch.float64)
            reqs.append(dist.irecv(t, peer))
            recvs.append((t, ra, rb))

        def wait():
            for r in reqs:
                r.wait()
            for t, ra, rb in recvs:
                buf[ra:rb] = t.numpy()
        return wait

    out = D.iterate(s, xa, xb, iters, spmv_rows_factory(s, vals, offs), exchange)
    q.put((rank, s.r0, out[s.own_lo:s.own_hi].copy()))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_iteration_is_bitwise_equal(world):
    iters = 4
    want = run_single(iters)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([p[2] for p in sorted(parts)])
    assert got.shape == want.shape
    assert np.array_equal(got, want)


def test_partition_geometry():
    n, h = 1000, 37
    slices = [D.partition(n, h, r, 4) for r in range(4)]
    assert slices[0].r0 == 0 and slices[-1].r1 == n
    assert all(a.r1 == b.r0 for a, b in zip(slices, slices[1:]))
    for s in slices:
        lo, hi = s.interior()
        # interior rows never read the halo
        assert all(0 <= r + s.own_lo - h and r + s.own_lo + h < s.nwin or s.world == 1
                   for r in range(lo, hi) if s.rank not in (0, s.world - 1))
        for peer, (sa, sb), (ra, rb) in D.halo_plan(s):
            assert sb - sa == min(h, s.nloc)
            assert s.own_lo <= sa and sb <= s.own_hi
            assert (ra, rb) in [(0, s.own_lo), (s.own_hi, s.nwin)]


def _lpt_worker(rank, world, port, weights, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    mine = D.lpt_shard(weights, world, rank)
    got = [None] * world
    dist.all_gather_object(got, (rank, mine))
    q.put(got)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batch_sharding_covers_every_matrix_once(world):
    """Config 4 batch sharding: each rank derives its LPT shard locally; the
    gathered shards partition the corpus and respect Graham's 4/3 bound."""
    rng = np.random.default_rng(4)
    weights = list(np.exp(rng.uniform(np.log(5e4), np.log(1.3e8), 200)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_lpt_worker, args=(r, world, port, weights, q)) for r in range(world)]
    for p in procs:
        p.start()
    views = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = dict(views[0])
    assert all(dict(v) == shards for v in views)  # every rank saw the same partition
    flat = sorted(i for r in range(world) for i in shards[r])
    assert flat == list(range(len(weights)))
    loads = [sum(weights[i] for i in shards[r]) for r in range(world)]
    assert max(loads) <= 4 / 3 * max(sum(weights) / world, max(weights)) + 1e-6


class _StubDistLib:
    """so_dist_* stand-in: create/handle succeed except on `fail_rank`, where
    the step named by `fail_at` returns an error (as a rank whose GPU cannot
    map its peers would)."""

    def __init__(self, rank, fail_rank, fail_at):
        self.rank, self.fail_rank, self.fail_at = rank, fail_rank, fail_at
        self.freed = 0

    def _st(self, step):
        return 7 if (self.rank == self.fail_rank and step == self.fail_at) else 0

    def so_dist_create(self, m, kind, rank, world, st, halo, out):
        out._obj.value = 1234
        return self._st("create")

    def so_dist_handle(self, h, buf):
        buf.raw = bytes([self.rank]) * 64
        return self._st("handle")

    def so_dist_connect(self, h, arr):
        return self._st("connect")

    def so_last_error(self):
        return f"stub failure on rank {self.rank}".encode()

    def so_dist_free(self, h):
        self.freed += 1


def _setup_fail_worker(rank, world, port, fail_rank, fail_at, q):
    from unittest import mock

    from paper_2303_05098_b200 import _capi
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    lib = _StubDistLib(rank, fail_rank, fail_at)

    class _M:
        _h = None
    with mock.patch.object(_capi, "lib", lambda: lib):
        try:
            D.DistIteration(_M(), D.HALO, rank, world, D.row_starts(60, world), 2, dist.all_gather_object)
            outcome = "ok"
        except D.DistSetupError as e:
            outcome = str(e)
    dist.barrier()  # every rank got here: nobody is stuck in a collective
    q.put((rank, outcome, lib.freed))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_at", ["create", "handle", "connect", None])
def test_dist_setup_failure_is_seen_by_every_rank(fail_at):
    """A so_dist setup failure on one rank raises DistSetupError on EVERY
    rank (so bench.py falls back to NCCL on all of them together) instead of
    leaving the healthy ranks blocked in all_gather_object."""
    world, fail_rank = 3, 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_setup_fail_worker, args=(r, world, port, fail_rank, fail_at, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, outcome, freed in got:
        if fail_at is None:
            assert outcome == "ok" and freed == 0
        else:
            assert "stub failure on rank 1" in outcome or "could not export" in outcome, outcome
            # whatever this rank created is freed again
            assert freed == (0 if (rank == fail_rank and fail_at == "create") else 1)
