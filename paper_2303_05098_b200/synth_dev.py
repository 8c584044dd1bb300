"""Device-side synthetic matrix generators (config 4 corpus, config 5 slices).

Input generation only -- torch on the GPU builds canonical CSR arrays
(int64 row_ptr, int32 col, f64 val) that are imported with
``DeviceMatrix.csr_device`` (a D2D copy into the library's own layout).
Nothing here is on a timed path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch


@dataclass
class DevCSR:
    nrows: int
    ncols: int
    row_ptr: torch.Tensor  # int64 [n+1]
    col: torch.Tensor      # int32 [z]
    val: torch.Tensor      # f64 [z]
    family: str = ""

    @property
    def nnz(self):
        return int(self.val.numel())

    def to_device_matrix(self):
        from .device import DeviceMatrix
        # the import copies on the library's stream: the producing torch work
        # must be complete first
        torch.cuda.synchronize()
        return DeviceMatrix.csr_device(self.nrows, self.ncols, self.nnz, self.row_ptr.data_ptr(),
                                       self.col.data_ptr(), self.val.data_ptr())


def _values(gen, z, dev):
    v = 0.5 + 1.5 * torch.rand(z, generator=gen, device=dev, dtype=torch.float64)
    s = torch.randint(0, 2, (z,), generator=gen, device=dev)
    return torch.where(s == 1, -v, v)


def _from_mask(n, m, cols, ok, gen):
    """cols/ok: [n, k] candidate columns (ascending per row) and validity."""
    dev = cols.device
    lens = ok.sum(dim=1)
    rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(lens, 0)
    col = cols[ok].to(torch.int32)
    return DevCSR(n, m, rp, col, _values(gen, col.numel(), dev))


def offsets_matrix(n, offsets, seed, dev="cuda", family="banded"):
    """Diagonals at the given offsets fully populated (clipped)."""
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    offs = torch.tensor(sorted(set(int(o) for o in offsets)), dtype=torch.int64, device=dev)
    i = torch.arange(n, dtype=torch.int64, device=dev)[:, None]
    cols = i + offs[None, :]
    ok = (cols >= 0) & (cols < n)
    out = _from_mask(n, n, cols, ok, gen)
    out.family = family
    return out


def stencil(g, dims=2, points=5, seed=0, dev="cuda"):
    """2-D 5/9-point or 3-D 7/27-point stencil on a g^dims grid."""
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    n = g ** dims
    i = torch.arange(n, dtype=torch.int64, device=dev)
    coords = []
    rem = i
    for _ in range(dims):
        coords.append(rem % g)
        rem = rem // g
    nbs = []
    rng = (-1, 0, 1)
    import itertools
    for d in itertools.product(rng, repeat=dims):
        nz = sum(abs(t) for t in d)
        if points in (5, 7) and nz > 1:
            continue
        nbs.append(d)
    strides = [g ** k for k in range(dims)]
    nbs.sort(key=lambda d: sum(t * s for t, s in zip(d, strides)))
    cols, oks = [], []
    for d in nbs:
        off = sum(t * s for t, s in zip(d, strides))
        ok = torch.ones(n, dtype=torch.bool, device=dev)
        for k, t in enumerate(d):
            c = coords[k] + t
            ok &= (c >= 0) & (c < g)
        cols.append(i + off)
        oks.append(ok)
    out = _from_mask(n, n, torch.stack(cols, 1), torch.stack(oks, 1), gen)
    out.family = f"stencil{dims}d{points}"
    return out


def _dedup(n, m, r, c, gen):
    key = r * m + c
    key = torch.unique(key)  # sorted
    rows = key // m
    cols = (key % m).to(torch.int32)
    rp = torch.zeros(n + 1, dtype=torch.int64, device=key.device)
    rp[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    return DevCSR(n, m, rp, cols, _values(gen, cols.numel(), key.device))


def uniform_random(n, degree, seed, dev="cuda"):
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    e = n * degree
    r = torch.randint(0, n, (e,), generator=gen, device=dev)
    c = torch.randint(0, n, (e,), generator=gen, device=dev)
    out = _dedup(n, n, r, c, gen)
    out.family = "uniform"
    return out


def rmat(n, degree, seed, dev="cuda", a=0.57, b=0.19, c=0.19):
    """R-MAT on the next power of two >= n, rows/cols folded back into [0, n)."""
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    scale = max(1, math.ceil(math.log2(n)))
    e = n * degree
    r = torch.zeros(e, dtype=torch.int64, device=dev)
    cc = torch.zeros(e, dtype=torch.int64, device=dev)
    for _ in range(scale):
        p = torch.rand(e, generator=gen, device=dev)
        q = (p >= a).to(torch.int64) + (p >= a + b).to(torch.int64) + (p >= a + b + c).to(torch.int64)
        r = 2 * r + (q >> 1)
        cc = 2 * cc + (q & 1)
    r %= n
    cc %= n
    out = _dedup(n, n, r, cc, gen)
    out.family = "powerlaw"
    return out


FAMILIES = ("stencil", "banded", "uniform", "powerlaw")


def corpus_spec(i, base_seed=4, nmin=10_000, nmax=5_000_000):
    """Deterministic spec of matrix i of the config-4 batch:
    500 each of stencil / banded / uniform-random / power-law, n log-uniform."""
    rng = np.random.default_rng([base_seed, i])
    fam = FAMILIES[i % 4]
    n = int(round(math.exp(rng.uniform(math.log(nmin), math.log(nmax)))))
    spec = {"id": i, "family": fam, "n": n, "seed": int(rng.integers(1 << 31))}
    if fam == "stencil":
        kind = ("2d5", "2d9", "3d7", "3d27")[int(rng.integers(4))]
        dims, pts = int(kind[0]), int(kind[2:])
        spec.update(dims=dims, points=pts, g=max(3, int(round(n ** (1.0 / dims)))))
    elif fam == "banded":
        nd = int(rng.integers(3, 28))
        bw = int(rng.integers(nd // 2, 4 * nd + 1))
        offs = set([0])
        while len(offs) < nd:
            offs.add(int(rng.integers(-bw, bw + 1)))
        spec.update(offsets=sorted(offs))
    elif fam == "uniform":
        spec.update(degree=int(rng.integers(4, 33)))
    else:
        spec.update(degree=int(rng.integers(4, 33)))
    return spec


def build(spec, dev="cuda"):
    fam = spec["family"]
    if fam == "stencil":
        return stencil(spec["g"], spec["dims"], spec["points"], spec["seed"], dev)
    if fam == "banded":
        return offsets_matrix(spec["n"], spec["offsets"], spec["seed"], dev)
    if fam == "uniform":
        return uniform_random(spec["n"], spec["degree"], spec["seed"], dev)
    return rmat(spec["n"], spec["degree"], spec["seed"], dev)


def nnz_estimate(spec):
    fam = spec["family"]
    if fam == "stencil":
        return spec["g"] ** spec["dims"] * spec["points"]
    if fam == "banded":
        return spec["n"] * len(spec["offsets"])
    return spec["n"] * spec["degree"]
