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


# ------------------------------------------------------ fused peer-memory halo

class PeerWindows:
    """The two x windows and the two halo flags of this rank in peer-shareable
    device memory (so_ipc_alloc), plus the neighbours' windows and flags
    mapped into this process (so_ipc_open: NVLink peer memory on an 8xB200
    node; plain device memory when ranks share one GPU).

    flags[0] is written by the left neighbour (my left halo is complete for
    iteration value-1), flags[1] by the right neighbour.  Handles travel once
    through `all_gather_object` (any torch.distributed backend)."""

    def __init__(self, s: Slice, all_gather_object):
        import ctypes as C

        from . import _capi as A
        if s.world > 1 and s.nloc < 2 * s.h:
            raise ValueError("fused halo exchange needs >= 2h owned rows per rank")
        self.s = s
        self._lib = A.lib()
        self._own = []

        def alloc(nbytes):
            p, h = C.c_void_p(), C.create_string_buffer(64)
            self._check(self._lib.so_ipc_alloc(nbytes, C.byref(p), h))
            self._own.append(p.value)
            return p.value, h.raw

        self.buf, hb = zip(*[alloc(8 * s.nwin) for _ in range(2)])
        self.flags, hf = alloc(16)
        self.tickets, _ = alloc(16)
        infos = [None] * s.world
        all_gather_object(infos, (s.rank, s.w0, list(hb), hf))
        self.peer = {}
        self._opened = []
        for nb in (s.rank - 1, s.rank + 1):
            if 0 <= nb < s.world:
                _, w0, bh, fh = infos[nb]
                ptrs = []
                for h in (*bh, fh):
                    p = C.c_void_p()
                    self._check(self._lib.so_ipc_open(h, C.byref(p)))
                    self._opened.append(p.value)
                    ptrs.append(p.value)
                self.peer[nb] = {"w0": w0, "buf": ptrs[:2], "flags": ptrs[2]}
        self.it = 0  # iterations completed (flag values are monotone)

    def _check(self, st):
        if st != 0:
            raise RuntimeError(self._lib.so_last_error().decode(errors="replace"))

    def tensor(self, k):
        """torch view (zero-copy, __cuda_array_interface__) of window k."""
        import torch

        class _View:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                                  "version": 3, "strides": None}
        return torch.as_tensor(_View(self.buf[k], self.s.nwin), device="cuda")

    def iterate(self, m, iters, stream):
        """`iters` steps of x <- A x on the windows, halo rows pushed to the
        neighbours by the multiply itself (so_spmv_rows_push), no collective.
        Returns the index of the window holding the last iterate."""
        import ctypes as C
        s, lib = self.s, self._lib
        lo, hi = s.interior()
        sp = C.c_void_p(stream)
        for _ in range(iters):
            it = self.it
            cur, nxt = self.buf[it % 2], self.buf[(it + 1) % 2]
            y = nxt + 8 * s.own_lo
            # my halo of `cur` was pushed by the neighbours during iteration it-1
            if s.rank > 0:
                self._check(lib.so_wait_flag(C.c_void_p(self.flags), it, sp))
            if s.rank < s.world - 1:
                self._check(lib.so_wait_flag(C.c_void_p(self.flags + 8), it, sp))
            if s.rank > 0:  # first h rows -> left neighbour's right halo
                p = self.peer[s.rank - 1]
                remote = p["buf"][(it + 1) % 2] + 8 * (s.r0 - p["w0"])
                self._check(lib.so_spmv_rows_push(m._h, C.c_void_p(cur), C.c_void_p(y), 0, lo,
                                                  C.c_void_p(remote), C.c_void_p(self.tickets),
                                                  C.c_void_p(p["flags"] + 8), it + 1, sp))
            if s.rank < s.world - 1:  # last h rows -> right neighbour's left halo
                p = self.peer[s.rank + 1]
                remote = p["buf"][(it + 1) % 2] + 8 * (s.r0 + hi - p["w0"])
                self._check(lib.so_spmv_rows_push(m._h, C.c_void_p(cur), C.c_void_p(y), hi, s.nloc,
                                                  C.c_void_p(remote), C.c_void_p(self.tickets + 4),
                                                  C.c_void_p(p["flags"]), it + 1, sp))
            if hi > lo:
                self._check(lib.so_spmv_device_rows(m._h, C.c_void_p(cur), C.c_void_p(y), lo, hi, sp))
            self.it += 1
        return self.it % 2

    def timeouts(self):
        """Halo waits that gave up (a neighbour never published): nonzero means
        the iterate is invalid (so_wait_flag_timeouts)."""
        return int(self._lib.so_wait_flag_timeouts())

    def close(self):
        for p in self._opened:
            self._lib.so_ipc_close(p)
        for p in self._own:
            self._lib.so_ipc_free(p)
        self._opened, self._own = [], []
