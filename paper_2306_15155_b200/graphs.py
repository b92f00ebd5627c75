"""Synthetic graphs.

* The reference's small bundled generators (path / star / grid / power-law /
  random; gnncompose/graphs.py:14-107), restated so the same seeds give the
  same graphs.
* Exact-nnz generators for the BASELINE shapes: uniform and
  RMAT(0.57, 0.19, 0.19, 0.05).  Candidate edges are a pure function of
  (seed, counter) through a splitmix64 hash written in torch integer ops, so
  the CPU (tests) and the GPU (bench) produce identical graphs.  The graph is
  the set of the first E distinct undirected pairs (u != v) in counter order,
  symmetrised: nnz(A) = 2E exactly, no self loops, unit values.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .sparse import CsrMatrix, default_device

# ---------------------------------------------------------------------------
# reference generators (gnncompose/graphs.py)
# ---------------------------------------------------------------------------


def _from_undirected_edges(n: int, src, dst, device=None) -> CsrMatrix:
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    a = CsrMatrix.from_coo(n, n, np.concatenate((src, dst)), np.concatenate((dst, src)),
                           np.ones(2 * src.size), sum_duplicates=True, device=device)
    return a.with_values(torch.ones(a.nnz, device=a.device))  # duplicates collapse to 1


def path_graph(n: int, device=None) -> CsrMatrix:
    if n < 1:
        raise ValueError("path_graph needs n >= 1")
    i = np.arange(n - 1, dtype=np.int64)
    return _from_undirected_edges(n, i, i + 1, device)


def star_graph(n: int, device=None) -> CsrMatrix:
    if n < 2:
        raise ValueError("star_graph needs n >= 2")
    return _from_undirected_edges(n, np.zeros(n - 1, dtype=np.int64), np.arange(1, n), device)


def grid_graph(rows: int, cols: int, device=None) -> CsrMatrix:
    if rows < 1 or cols < 1:
        raise ValueError("grid_graph needs positive dimensions")
    idx = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    src = np.concatenate((idx[:, :-1].ravel(), idx[:-1, :].ravel()))
    dst = np.concatenate((idx[:, 1:].ravel(), idx[1:, :].ravel()))
    return _from_undirected_edges(rows * cols, src, dst, device)


def powerlaw_graph(n: int, m: int, seed: int = 0, device=None) -> CsrMatrix:
    """Preferential attachment with the repeated-endpoint trick; same draws as
    the reference for the same seed."""
    if n <= m or m < 1:
        raise ValueError("powerlaw_graph needs n > m >= 1")
    rng = np.random.default_rng(seed)
    src, dst = [], []
    ends = list(range(m + 1))
    for u in range(m):
        for v in range(u + 1, m + 1):
            src.append(u)
            dst.append(v)
    for u in range(m + 1, n):
        tg: set[int] = set()
        while len(tg) < m:
            tg.add(int(ends[rng.integers(len(ends))]))
        for v in tg:
            src.append(u)
            dst.append(v)
            ends.append(u)
            ends.append(v)
    return _from_undirected_edges(n, src, dst, device)


def random_graph(n: int, density: float, seed: int = 0, device=None) -> CsrMatrix:
    if n < 1:
        raise ValueError("random_graph needs n >= 1")
    if not 0.0 < density <= 1.0:
        raise ValueError("density must be in (0, 1]")
    rng = np.random.default_rng(seed)
    e = max(1, int(round(density * n * n / 2)))
    s = rng.integers(0, n, size=e, dtype=np.int64)
    d = rng.integers(0, n, size=e, dtype=np.int64)
    keep = s != d
    return _from_undirected_edges(n, s[keep], d[keep], device)


BUNDLED_GRAPHS = {
    "path4096": lambda device=None: path_graph(4096, device),
    "star2048": lambda device=None: star_graph(2048, device),
    "grid64x64": lambda device=None: grid_graph(64, 64, device),
    "powerlaw4096": lambda device=None: powerlaw_graph(4096, 8, seed=7, device=device),
}


def bundled_graphs(device=None) -> list[tuple[str, CsrMatrix]]:
    return [(k, f(device)) for k, f in BUNDLED_GRAPHS.items()]


# ---------------------------------------------------------------------------
# counter-based hashing (identical on CPU and GPU)
# ---------------------------------------------------------------------------

_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    x &= _M64
    return x - (1 << 64) if x >= 1 << 63 else x


_C1, _C2, _GOLD = _s64(0xBF58476D1CE4E5B9), _s64(0x94D049BB133111EB), _s64(0x9E3779B97F4A7C15)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 (two's complement) values."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + _GOLD
    z = (z ^ _srl(z, 30)) * _C1
    z = (z ^ _srl(z, 27)) * _C2
    return z ^ _srl(z, 31)


def _splitmix64_int(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _unit(z: torch.Tensor) -> torch.Tensor:
    """Top 53 bits -> float64 in [0, 1) (exact on every device)."""
    return _srl(z, 11).double() * (1.0 / (1 << 53))


RMAT_PROBS = (0.57, 0.19, 0.19, 0.05)


def _candidates(kind: str, n: int, seed_key: int, start: int, count: int, device,
                probs=RMAT_PROBS) -> tuple[torch.Tensor, torch.Tensor]:
    ctr = torch.arange(start, start + count, dtype=torch.int64, device=device)
    if kind == "uniform":
        u = torch.remainder(_srl(splitmix64((ctr << 1) ^ seed_key), 1), n)
        v = torch.remainder(_srl(splitmix64(((ctr << 1) | 1) ^ seed_key), 1), n)
        return u, v
    if kind != "rmat":
        raise ValueError(f"unknown graph kind {kind!r}")
    levels = max(1, math.ceil(math.log2(n)))
    a, b, c, _ = probs
    t1, t2, t3 = a, a + b, a + b + c
    u = torch.zeros(count, dtype=torch.int64, device=device)
    v = torch.zeros(count, dtype=torch.int64, device=device)
    base = ctr << 6
    for lvl in range(levels):
        r = _unit(splitmix64((base | lvl) ^ seed_key))
        ubit = (r >= t2).long()  # quadrants 2, 3: lower half
        vbit = ((r >= t1) & (r < t2)).long() | (r >= t3).long()  # quadrants 1, 3: right half
        u = (u << 1) | ubit
        v = (v << 1) | vbit
    return u, v


def synthetic_graph(kind: str, n: int, nnz: int, seed: int = 0, device=None,
                    chunk: int = 1 << 25, max_candidates: int = 1 << 34) -> CsrMatrix:
    """Symmetric unit-valued graph with exactly ``nnz`` stored entries
    (``nnz`` even; nnz/2 distinct undirected pairs, no self loops)."""
    if nnz % 2 or nnz < 0:
        raise ValueError("nnz must be even and non-negative")
    target = nnz // 2
    if target > n * (n - 1) // 2:
        raise ValueError("more edges than node pairs")
    dev = torch.device(device) if device is not None else default_device()
    seed_key = _s64(_splitmix64_int(seed * 0x100000001B3 + 0x5BD1E995))
    keys = torch.empty(0, dtype=torch.int64, device=dev)  # sorted accepted pair keys
    start = 0
    step = min(chunk, max(4096, 2 * target))
    while keys.numel() < target:
        if start >= max_candidates:
            raise RuntimeError(f"{kind} generator: {keys.numel()} of {target} distinct pairs after "
                               f"{start} candidates")
        u, v = _candidates(kind, n, seed_key, start, step, dev)
        start += step
        step = min(chunk, 2 * step)
        ok = (u < n) & (v < n) & (u != v)
        lo, hi = torch.minimum(u, v)[ok], torch.maximum(u, v)[ok]
        ck = lo * n + hi  # candidate keys in counter order
        if keys.numel():
            pos = torch.searchsorted(keys, ck).clamp_max(keys.numel() - 1)
            ck = ck[keys[pos] != ck]
        if ck.numel() == 0:
            continue
        sk, order = torch.sort(ck, stable=True)
        first = torch.ones_like(sk, dtype=torch.bool)
        first[1:] = sk[1:] != sk[:-1]
        new_keys, new_pos = sk[first], order[first]
        need = target - keys.numel()
        if new_keys.numel() > need:  # keep the earliest in counter order
            keep = torch.sort(new_pos).indices[:need]
            new_keys = new_keys[keep]
        keys = torch.sort(torch.cat([keys, new_keys])).values
    lo, hi = keys // n, keys % n
    rows = torch.cat([lo, hi])
    cols = torch.cat([hi, lo])
    ckey, order = torch.sort(rows * n + cols)
    cols = cols[order]
    counts = torch.bincount(ckey // n, minlength=n)
    row_ptr = torch.cat([counts.new_zeros(1), torch.cumsum(counts, 0)])
    g = CsrMatrix(n, n, row_ptr, cols, torch.ones(cols.numel(), device=dev), validate=False,
                  device=dev)
    g._unit = True
    return g


# ---------------------------------------------------------------------------
# the BASELINE shapes (nnz = stored, both directions)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class GraphShape:
    name: str
    kind: str
    n: int
    nnz: int


SHAPES = {
    "cora": GraphShape("cora", "uniform", 2_708, 10_556),
    "arxiv": GraphShape("arxiv", "rmat", 169_343, 2_332_486),
    "reddit": GraphShape("reddit", "rmat", 232_965, 114_615_892),
    "products": GraphShape("products", "rmat", 2_449_029, 123_718_280),
}


def shape_graph(name: str, seed: int = 0, device=None) -> CsrMatrix:
    s = SHAPES[name]
    return synthetic_graph(s.kind, s.n, s.nnz, seed=seed, device=device)
