"""Row-partitioned iterated SpMV with halo exchange (config 5).

Rank p of P owns rows [r0, r1) = [p*n/P, (p+1)*n/P) of a banded / stencil
DIA matrix and keeps x on the window [w0, w1) = [r0-h, r1+h) clipped to
[0, n), where h = max |offset| (g^2+g+1 for the 27-point stencil).  Every
iteration computes y on the owned rows straight into the next x window and
exchanges the h-row halos with p-1 / p+1 (point-to-point; NCCL over NVLink on
the GPU path, gloo in the CPU tests).  Rows whose window lies inside the owned
range (interior) need no halo, so the boundary rows are computed first, the
exchange is started, and the interior overlaps it.

The row partition does not change any row's summation order, so the P-rank
result is bitwise equal to the 1-rank result (tests/test_dist_host.py).

This module is pure plumbing: the multiply is a callable (the sm_100a DIA
kernel through ``so_spmv_device_rows`` on the GPU path).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Slice:
    n: int      # global rows = cols
    h: int      # halo width = max |offset|
    rank: int
    world: int
    r0: int     # owned rows [r0, r1)
    r1: int
    w0: int     # x window [w0, w1)
    w1: int

    @property
    def own_lo(self):  # owned rows inside the window
        return self.r0 - self.w0

    @property
    def own_hi(self):
        return self.r1 - self.w0

    @property
    def nloc(self):
        return self.r1 - self.r0

    @property
    def nwin(self):
        return self.w1 - self.w0

    def interior(self):
        """local rows whose band lies inside the owned x range"""
        lo = min(self.h, self.nloc) if self.rank > 0 else 0
        hi = max(self.nloc - self.h, lo) if self.rank < self.world - 1 else self.nloc
        return lo, hi


def partition(n: int, h: int, rank: int, world: int) -> Slice:
    r0 = n * rank // world
    r1 = n * (rank + 1) // world
    if world > 1 and h > n // world:
        raise ValueError("halo wider than a rank's row slice: use fewer ranks")
    return Slice(n, h, rank, world, r0, r1, max(0, r0 - h), min(n, r1 + h))


def local_offsets(offsets, s: Slice):
    """DIA offsets of the local (nloc x nwin) block: col_local = row_local + off + (r0 - w0)."""
    return [int(o) + (s.r0 - s.w0) for o in offsets]


def halo_plan(s: Slice):
    """(peer, send window range, recv window range) for each neighbour."""
    plan = []
    if s.rank > 0:  # left neighbour owns [.., r0): it needs my first h rows
        k = min(s.h, s.nloc)
        plan.append((s.rank - 1, (s.own_lo, s.own_lo + k), (0, s.own_lo)))
    if s.rank < s.world - 1:
        k = min(s.h, s.nloc)
        plan.append((s.rank + 1, (s.own_hi - k, s.own_hi), (s.own_hi, s.nwin)))
    return plan


def iterate(s: Slice, x_cur, x_next, iters, spmv_rows, exchange, copy=None):
    """Run `iters` y = A x steps in place on the window buffers.

    spmv_rows(x_win, y_out_window, lo, hi): y_out_window[own_lo+lo : own_lo+hi]
        = (A x)[local rows lo:hi]
    exchange(buf, plan) -> waitable: halo exchange on window buffer `buf`.
    Returns the buffer holding the last iterate."""
    lo, hi = s.interior()
    plan = halo_plan(s)
    for _ in range(iters):
        # boundary rows first: they are what the neighbours need
        if lo > 0:
            spmv_rows(x_cur, x_next, 0, lo)
        if hi < s.nloc:
            spmv_rows(x_cur, x_next, hi, s.nloc)
        pending = exchange(x_next, plan)
        spmv_rows(x_cur, x_next, lo, hi)  # interior overlaps the exchange
        if pending is not None:
            pending()
        x_cur, x_next = x_next, x_cur
    return x_cur


# ------------------------------------------------ batches of independent matrices

def lpt_shard(weights, world: int, rank: int):
    """Greedy longest-processing-time assignment of independent items (config
    4: matrices weighted by their nnz) to `world` ranks; returns this rank's
    item indices in ascending order.  Deterministic (ties -> lowest index /
    rank), so every rank computes the same partition without communication;
    the largest load is at most 4/3 of optimal (Graham's bound)."""
    loads = [0.0] * world
    mine = []
    for i in sorted(range(len(weights)), key=lambda i: (-weights[i], i)):
        r = min(range(world), key=lambda k: (loads[k], k))
        loads[r] += weights[i]
        if r == rank:
            mine.append(i)
    return sorted(mine)


# ------------------------------------------- native iteration (so_dist_* C-ABI)

HALO, ALLGATHER = 0, 1  # SO_DIST_HALO, SO_DIST_ALLGATHER


class DistSetupError(RuntimeError):
    """so_dist setup failed on at least one rank (raised on every rank)."""


def row_starts(n: int, world: int):
    """The partition of `partition` as the row_starts array of so_dist_create."""
    return [n * q // world for q in range(world + 1)]


class DistIteration:
    """Row-partitioned x <- A x across ranks through the library's so_dist_*
    entry points (csrc/dist.cu): the x exchange is done by the library's own
    kernels over peer memory (HALO: boundary rows pushed into the neighbours'
    windows by the multiply; ALLGATHER: new rows stored into every peer's x),
    no collective on the data path.  The IPC handles travel once through
    `all_gather_object` (any torch.distributed backend).

    Setup is collective-safe: every rank reaches both `all_gather_object`
    calls whatever fails locally (create, handle export, peer mapping), and a
    failure on ANY rank raises `DistSetupError` on EVERY rank (after freeing
    what was built), so callers can fall back together instead of one rank
    hanging in a collective the others never enter."""

    def __init__(self, m, kind, rank, world, starts, halo, all_gather_object):
        import ctypes as C

        from . import _capi as A
        self._lib = A.lib()
        self._C = C
        self._h = None
        self.m = m  # the so_dist borrows the matrix: keep it alive
        st = (C.c_int64 * (world + 1))(*starts)
        err = None
        mine = C.create_string_buffer(64)
        try:
            h = C.c_void_p()
            self._check(self._lib.so_dist_create(m._h, kind, rank, world, st, int(halo), C.byref(h)))
            self._h = h
            self._check(self._lib.so_dist_handle(self._h, mine))
        except RuntimeError as e:
            err = f"rank {rank}: {e}"
        infos = [None] * world
        all_gather_object(infos, None if err else mine.raw)
        bad = [i for i, v in enumerate(infos) if v is None]
        if not err and bad:
            err = f"rank(s) {bad} could not export their x block"
        if not err:
            arr = C.create_string_buffer(b"".join(infos), 64 * world)
            try:
                self._check(self._lib.so_dist_connect(self._h, arr))
            except RuntimeError as e:
                err = f"rank {rank}: {e}"
        errs = [None] * world
        all_gather_object(errs, err)
        errs = [e for e in errs if e]
        if errs:
            self.close()
            raise DistSetupError("; ".join(errs))

    def _check(self, st):
        if st != 0:
            raise RuntimeError(self._lib.so_last_error().decode(errors="replace"))

    def x(self, which=-1):
        """(device pointer, global offset, length) of x buffer `which` (-1: latest iterate)."""
        C = self._C
        p, off, ln = C.c_void_p(), C.c_int64(), C.c_int64()
        self._check(self._lib.so_dist_x(self._h, int(which), C.byref(p), C.byref(off), C.byref(ln)))
        return p.value, off.value, ln.value

    def tensor(self, which=-1):
        """torch view (zero-copy, __cuda_array_interface__) of an x buffer."""
        import torch
        ptr, _, ln = self.x(which)

        class _View:
            def __init__(self):
                self.__cuda_array_interface__ = {"shape": (ln,), "typestr": "<f8", "data": (ptr, False),
                                                  "version": 3, "strides": None}
        return torch.as_tensor(_View(), device="cuda")

    def iterate(self, iters, stream=0):
        self._check(self._lib.so_dist_iterate(self._h, int(iters), self._C.c_void_p(stream)))

    def timeouts(self):
        return int(self._lib.so_dist_timeouts())

    def close(self):
        if self._h:
            self._lib.so_dist_free(self._h)
            self._h = None


class _NativeIterator:
    """bench adapter: the so_dist HALO iteration."""

    def __init__(self, s: Slice, m, dist, stream):
        self.s, self.stream = s, stream
        self.it = DistIteration(m, HALO, s.rank, s.world, row_starts(s.n, s.world), s.h, dist.all_gather_object)

    def load_x(self, fn):
        # the buffer the next iteration reads (halo cells included)
        self.it.tensor(-1).copy_(fn(self.s.w0, self.s.w1))

    def run(self, iters):
        self.it.iterate(iters, self.stream.cuda_stream)

    def owned(self):
        return self.it.tensor(-1)[self.s.own_lo:self.s.own_hi]

    def checksum(self):
        return owned_checksum(self.owned(), self.s)

    def timeouts(self):
        return self.it.timeouts()

    def close(self):
        self.it.close()


class _NcclIterator:
    """bench adapter: `iterate` with torch.distributed isend/irecv halos
    (NCCL point-to-point) after the boundary rows."""

    def __init__(self, s: Slice, m, dist, stream):
        import torch
        self.s, self.m, self.dist, self.stream = s, m, dist, stream
        self.xa = torch.zeros(s.nwin, dtype=torch.float64, device="cuda")
        self.xb = torch.zeros_like(self.xa)

    def load_x(self, fn):
        self.xa.copy_(fn(self.s.w0, self.s.w1))

    def run(self, iters):
        s, m, dist, st = self.s, self.m, self.dist, self.stream

        def spmv_rows(xw, yw, lo, hi):
            m.spmv_device_rows(xw.data_ptr(), yw.data_ptr() + 8 * s.own_lo, lo, hi, st.cuda_stream)

        def exchange(buf, plan):
            reqs = []
            for peer, (sa, sb), (ra, rb) in plan:
                reqs.append(dist.isend(buf[sa:sb], peer))
                reqs.append(dist.irecv(buf[ra:rb], peer))
            return lambda: [r.wait() for r in reqs]

        out = iterate(s, self.xa, self.xb, iters, spmv_rows, exchange)
        if out is not self.xa:
            self.xa, self.xb = self.xb, self.xa

    def owned(self):
        return self.xa[self.s.own_lo:self.s.own_hi]

    def checksum(self):
        return owned_checksum(self.owned(), self.s)

    def timeouts(self):
        return 0

    def close(self):
        pass


def owned_checksum(owned, s: Slice):
    """Order-independent bitwise checksum of the whole iterate:
    sum_i (2 i + 1) * bits(x_i) mod 2^64 over global rows i (wrapping int64
    arithmetic, a commutative ring), so every partition of the same iterate
    gives the same number and any changed bit changes it."""
    import torch
    import torch.distributed as dist
    bits = owned.contiguous().view(torch.int64)
    idx = torch.arange(s.r0, s.r1, dtype=torch.int64, device=owned.device) * 2 + 1
    local = (bits * idx).sum().reshape(1)
    if dist.is_available() and dist.is_initialized() and s.world > 1:
        if dist.get_backend() == "gloo":
            local = local.cpu()
        dist.all_reduce(local)
    return int(local.item()) & ((1 << 64) - 1)


def make_iterator(s: Slice, m, dist, exchange, stream):
    """The config-5 iteration for bench.py: 'p2p' -> the native fused-halo
    so_dist iteration, 'nccl' -> NCCL point-to-point halos.  If the peer
    mapping cannot be set up on some rank (no peer access between the
    devices, IPC refused), every rank falls back to NCCL together; the
    returned iterator's `exchange` / `fallback` say what ran and why."""
    if exchange == "p2p":
        try:
            it = _NativeIterator(s, m, dist, stream)
            it.exchange, it.fallback = "p2p", None
            return it
        except DistSetupError as e:
            it = _NcclIterator(s, m, dist, stream)
            it.exchange, it.fallback = "nccl", f"p2p setup failed: {e}"[:300]
            return it
    it = _NcclIterator(s, m, dist, stream)
    it.exchange, it.fallback = "nccl", None
    return it
