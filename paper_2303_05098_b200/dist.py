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
