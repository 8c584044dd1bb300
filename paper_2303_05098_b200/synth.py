"""Synthetic matrices of the shapes BASELINE.json names.

Every generator returns a canonical CSR in the reference host layout
(int64 row_ptr / col, float64 values; rows sorted, no duplicates), i.e. what
``from_coo(CooMatrix::from_triplets(...), CSR)`` would hold.  Values are
+-U(0.5, 2) (never zero, oracles.hpp:176-181) unless stated.  Large R-MAT
draws run through torch on the GPU when one is present (input generation
only -- not part of any timed path).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class HostCSR:
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self):
        return int(self.val.size)

    def coo_rows(self):
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_ptr))


def _values(rng: np.random.Generator, n: int) -> np.ndarray:
    v = rng.uniform(0.5, 2.0, n)
    sign = rng.integers(0, 2, n, dtype=np.int8)
    v[sign == 1] *= -1.0
    return v


def _from_offsets(n: int, m: int, offsets, rng) -> HostCSR:
    """All listed diagonals fully populated (clipped to the matrix)."""
    offs = np.asarray(sorted(offsets), dtype=np.int64)
    lens = np.zeros(n, dtype=np.int64)
    for o in offs:
        lo, hi = max(0, -o), min(n, m - o)
        if hi > lo:
            lens[lo:hi] += 1
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    col = np.empty(int(rp[-1]), dtype=np.int64)
    fill = rp[:-1].copy()
    for o in offs:  # ascending offsets => columns ascending within each row
        lo, hi = max(0, -o), min(n, m - o)
        if hi <= lo:
            continue
        rows = np.arange(lo, hi, dtype=np.int64)
        col[fill[lo:hi]] = rows + o
        fill[lo:hi] += 1
    return HostCSR(n, m, rp, col, _values(rng, col.size))


def laplacian_2d(g: int, seed: int = 1) -> HostCSR:
    """Config 1: 5-point stencil on a g x g row-major grid (z = 5n - 4g).

    Offsets {-g, -1, 0, 1, g}; the +-1 neighbours are removed at grid-row
    boundaries, so this is not a plain banded matrix."""
    n = g * g
    rng = np.random.default_rng(seed)
    i = np.arange(n, dtype=np.int64)
    x = i % g
    cols = np.stack([i - g, i - 1, i, i + 1, i + g], axis=1)
    ok = np.stack([i >= g, x > 0, np.ones(n, bool), x < g - 1, i < n - g], axis=1)
    lens = ok.sum(axis=1)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    col = cols[ok]
    return HostCSR(n, n, rp, col, _values(rng, col.size))


def banded(n: int, half: int, seed: int = 2) -> HostCSR:
    """Config 2: every diagonal in [-half, half] fully populated
    (27 diagonals for half = 13; z = (2h+1) n - h (h+1))."""
    return _from_offsets(n, n, range(-half, half + 1), np.random.default_rng(seed))


def stencil_3d(g: int, points: int = 27, seed: int = 5) -> HostCSR:
    """3-D 7- or 27-point stencil on a g^3 grid (config 5 shape, small g)."""
    n = g ** 3
    rng = np.random.default_rng(seed)
    i = np.arange(n, dtype=np.int64)
    z, y, x = i // (g * g), (i // g) % g, i % g
    nb = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if points == 7 and abs(dz) + abs(dy) + abs(dx) > 1:
                    continue
                nb.append((dz, dy, dx))
    nb.sort(key=lambda t: t[0] * g * g + t[1] * g + t[2])
    cols = np.stack([i + dz * g * g + dy * g + dx for dz, dy, dx in nb], axis=1)
    ok = np.stack([(z + dz >= 0) & (z + dz < g) & (y + dy >= 0) & (y + dy < g) & (x + dx >= 0) & (x + dx < g)
                   for dz, dy, dx in nb], axis=1)
    lens = ok.sum(axis=1)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    col = cols[ok]
    return HostCSR(n, n, rp, col, _values(rng, col.size))


def _dedup(n: int, rows, cols, vals) -> HostCSR:
    key = rows * n + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    uniq, start = np.unique(key, return_index=True)
    summed = np.add.reduceat(vals, start) if vals.size else vals
    r = uniq // n
    c = uniq % n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    np.cumsum(rp, out=rp)
    return HostCSR(n, n, rp, c.astype(np.int64), summed.astype(np.float64))


def rmat(scale: int, degree: int = 16, seed: int = 42, a=0.57, b=0.19, c=0.19) -> HostCSR:
    """Config 3: R-MAT power law, degree * 2^scale edge draws, duplicates summed.

    Per level p = U[0,1): quadrant 0 if p < a, 1 if < a+b, 2 if < a+b+c else 3;
    r = 2r + (q >> 1), c = 2c + (q & 1).  Values are dyadic +-(1 + k/8) so the
    duplicate sums are exact in any order."""
    n = 1 << scale
    e = degree * n
    try:
        import torch

        dev = "cuda" if torch.cuda.is_available() else "cpu"
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        r = torch.zeros(e, dtype=torch.int64, device=dev)
        cc = torch.zeros(e, dtype=torch.int64, device=dev)
        for _ in range(scale):
            p = torch.rand(e, generator=gen, device=dev)
            q = (p >= a).to(torch.int64) + (p >= a + b).to(torch.int64) + (p >= a + b + c).to(torch.int64)
            r = 2 * r + (q >> 1)
            cc = 2 * cc + (q & 1)
        k = torch.randint(0, 8, (e,), generator=gen, device=dev)
        s = torch.randint(0, 2, (e,), generator=gen, device=dev)
        v = (1.0 + k.double() / 8.0) * (1 - 2 * s).double()
        key = r * n + cc
        key, order = torch.sort(key)
        v = v[order]
        uniq, inv = torch.unique_consecutive(key, return_inverse=True)
        summed = torch.zeros(uniq.numel(), dtype=torch.float64, device=dev).index_add_(0, inv, v)
        rows = (uniq // n).cpu().numpy()
        cols = (uniq % n).cpu().numpy()
        vals = summed.cpu().numpy()
        rp = np.zeros(n + 1, dtype=np.int64)
        np.add.at(rp, rows + 1, 1)
        np.cumsum(rp, out=rp)
        return HostCSR(n, n, rp, cols.astype(np.int64), vals)
    except ImportError:
        rng = np.random.default_rng(seed)
        r = np.zeros(e, np.int64)
        cc = np.zeros(e, np.int64)
        for _ in range(scale):
            p = rng.random(e)
            q = (p >= a).astype(np.int64) + (p >= a + b) + (p >= a + b + c)
            r = 2 * r + (q >> 1)
            cc = 2 * cc + (q & 1)
        v = (1.0 + rng.integers(0, 8, e) / 8.0) * np.where(rng.integers(0, 2, e) == 1, -1.0, 1.0)
        return _dedup(n, r, cc, v)


def uniform_random(n: int, degree: int, seed: int = 4) -> HostCSR:
    """Uniform-random rows (avg degree `degree`), duplicates merged."""
    rng = np.random.default_rng(seed)
    e = n * degree
    rows = rng.integers(0, n, e, dtype=np.int64)
    cols = rng.integers(0, n, e, dtype=np.int64)
    v = (1.0 + rng.integers(0, 8, e) / 8.0) * np.where(rng.integers(0, 2, e) == 1, -1.0, 1.0)
    return _dedup(n, rows, cols, v)


def hyb_skewed(n: int, short: int = 16, long: int = 160, every: int = 100, seed: int = 6) -> HostCSR:
    """HYB-favourable evidence matrix (SURVEY.md §8d "favourable matrix per
    format"): every row holds `short` consecutive columns centred on the
    diagonal, except every `every`-th row (rows i with i % every == every//2)
    which holds `long`; windows are shifted inward at the edges so every row is
    full.  With the reference's default K_H = ceil(z/n) (formats.cpp:357-361)
    the short rows fill the ELL part and each long row overflows
    long - K_H entries into the COO part (16/160/100: K_H = 18, COO part 8 %)."""
    rng = np.random.default_rng(seed)
    lens = np.full(n, short, dtype=np.int64)
    lens[every // 2::every] = long
    lens = np.minimum(lens, n)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    start = np.clip(np.arange(n, dtype=np.int64) - lens // 2, 0, n - lens)
    col = start[rows] + (np.arange(rp[-1], dtype=np.int64) - rp[rows])
    return HostCSR(n, n, rp, col, _values(rng, col.size))
