"""TEST INFRASTRUCTURE — CPU oracle for the GCN/GAT composition hot path.

A restatement of the reference package ``gnncompose`` 0.1.0
(``/root/reference/pkg/src/gnncompose``) in numpy + a small C/OpenMP library
(``oracle/csrc/oracle_kernels.c``).  Float64 values and int64 indices, the
reference's own precision, so the oracle reproduces the reference bit for bit
on the kernels (same per-row, ascending-column accumulation order; no FMA
contraction) and to the last ulp on the BLAS calls (numpy's ``@`` is the same
OpenBLAS the reference calls).

The oracle is PINNED by ``tests/test_oracle_golden.py``: it is compared with
golden vectors that ``tests/golden/make_golden.py`` produced by importing the
reference itself.

Who may use this module: ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and the ``--impl reference`` arm) —
only as the checker or the timed CPU baseline.  The product package
``paper_2306_15155_b200`` never imports it; its CUDA path fails loudly when
the extension is missing.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import zlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> Path:
    """Compile liboracle.so (gcc, OpenMP, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        lib.oracle_spmm_f64.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, ctypes.c_int64, _f64p, _f64p]
        lib.oracle_sddmm_f64.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, ctypes.c_int64, _f64p, _f64p, _f64p]
        lib.oracle_edge_softmax_f64.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, ctypes.c_double, _f64p]
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_get_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def set_threads(n: int | None = None) -> int:
    """Pin the OpenMP pool (the reference's numba pool) and BLAS to ``n`` threads.

    Mirrors gnncompose/runtime.py:25-44 (configure_threads).
    """
    n = n or os.cpu_count() or 1
    _load().oracle_set_threads(int(n))
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=int(n))
    except ImportError:  # pragma: no cover
        pass
    return int(n)


def get_threads() -> int:
    return int(_load().oracle_get_threads())


def _p64(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def _pf(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_f64p)


# ---------------------------------------------------------------------------
# CSR container — reference gnncompose/sparse.py:43-188
# ---------------------------------------------------------------------------


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # int64
    col_idx: np.ndarray  # int64
    values: np.ndarray  # float64

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.col_idx.size)

    @property
    def has_unit_values(self) -> bool:  # sparse.py:70-72
        return bool(self.values.size == 0 or np.all(self.values == 1.0))

    def degrees(self) -> np.ndarray:  # sparse.py:163-165
        return np.diff(self.row_ptr)

    def row_of_nnz(self) -> np.ndarray:  # sparse.py:167-169
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), self.degrees())

    def with_values(self, values) -> "Csr":  # sparse.py:148-156
        return Csr(self.n_rows, self.n_cols, self.row_ptr, self.col_idx, values)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols))
        out[self.row_of_nnz(), self.col_idx] = self.values
        return out

    def take_rows(self, rows) -> "Csr":
        """Row-sampled sub-CSR (full columns) for parity at sizes where the
        full f64 oracle would not fit."""
        rows = np.asarray(rows, dtype=np.int64)
        lo, hi = self.row_ptr[rows], self.row_ptr[rows + 1]
        cnt = hi - lo
        rp = np.concatenate(([0], np.cumsum(cnt)))
        idx = np.repeat(lo - rp[:-1], cnt) + np.arange(rp[-1], dtype=np.int64)
        return Csr(rows.size, self.n_cols, rp, self.col_idx[idx], self.values[idx])


def from_coo(n_rows, n_cols, rows, cols, values, sum_duplicates=True) -> Csr:
    """reference gnncompose/sparse.py:120-146: lexsort by (row, col); duplicate
    coordinates summed with np.add.reduceat in sorted order."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, values = rows[order], cols[order], values[order]
    if sum_duplicates and rows.size:
        first = np.empty(rows.size, dtype=bool)
        first[0] = True
        first[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        starts = np.flatnonzero(first)
        values = np.add.reduceat(values, starts)
        rows, cols = rows[starts], cols[starts]
    row_ptr = np.concatenate(([0], np.cumsum(np.bincount(rows, minlength=n_rows))))
    return Csr(n_rows, n_cols, row_ptr, cols, values)


def undirected_unit_graph(n: int, src, dst) -> Csr:
    """reference gnncompose/graphs.py:14-22: symmetrise, dedup, unit values."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    a = from_coo(n, n, np.concatenate((src, dst)), np.concatenate((dst, src)),
                 np.ones(2 * src.size))
    return a.with_values(np.ones(a.nnz))


def add_self_loops(a: Csr) -> Csr:
    """reference gnncompose/sparse.py:303-324 (value 1.0 on missing diagonals;
    existing diagonal entries kept; idempotent)."""
    if a.n_rows != a.n_cols:
        raise ValueError("add_self_loops requires a square matrix")
    rows = a.row_of_nnz()
    has_diag = np.zeros(a.n_rows, dtype=bool)
    has_diag[rows[a.col_idx == rows]] = True
    missing = np.flatnonzero(~has_diag)
    if missing.size == 0:
        return a
    return from_coo(a.n_rows, a.n_cols, np.concatenate((rows, missing)),
                    np.concatenate((a.col_idx, missing)),
                    np.concatenate((a.values, np.ones(missing.size))), sum_duplicates=False)


def inv_sqrt_degrees(a: Csr) -> np.ndarray:
    """reference gnncompose/sparse.py:327-336 (structural degree ^ -1/2)."""
    deg = a.degrees()
    if np.any(deg == 0):
        raise ValueError("zero-degree row")
    return 1.0 / np.sqrt(deg.astype(np.float64))


# ---------------------------------------------------------------------------
# kernels — reference gnncompose/sparse.py:240-300
# ---------------------------------------------------------------------------


def _dense(b) -> np.ndarray:
    return np.ascontiguousarray(b, dtype=np.float64)


def spmm(a: Csr, b) -> np.ndarray:
    """reference sparse.py:240-247 → _spmm_kernel 196-205."""
    b = _dense(b)
    assert a.n_cols == b.shape[0]
    out = np.zeros((a.n_rows, b.shape[1]))
    _load().oracle_spmm_f64(a.n_rows, _p64(a.row_ptr), _p64(a.col_idx), _pf(a.values),
                            b.shape[1], _pf(b), _pf(out))
    return out


def spmm_unweighted(a: Csr, b) -> np.ndarray:
    """reference sparse.py:250-264 → _spmm_unweighted_kernel 208-219 (values never read)."""
    b = _dense(b)
    assert a.n_cols == b.shape[0]
    out = np.zeros((a.n_rows, b.shape[1]))
    _load().oracle_spmm_f64(a.n_rows, _p64(a.row_ptr), _p64(a.col_idx), None,
                            b.shape[1], _pf(b), _pf(out))
    return out


def sddmm(a: Csr, b, c) -> Csr:
    """reference sparse.py:267-282 → _sddmm_kernel 222-232."""
    b, c = _dense(b), _dense(c)
    assert b.shape[0] == a.n_rows and c.shape[0] == a.n_cols and b.shape[1] == c.shape[1]
    out = np.empty(a.nnz)
    _load().oracle_sddmm_f64(a.n_rows, _p64(a.row_ptr), _p64(a.col_idx), _pf(a.values),
                             b.shape[1], _pf(b), _pf(c), _pf(out))
    return a.with_values(out)


def gemm(a, b) -> np.ndarray:
    """reference sparse.py:285-291 (numpy/OpenBLAS a @ b)."""
    return _dense(a) @ _dense(b)


def scale_rows(d, b) -> np.ndarray:
    """reference sparse.py:294-300."""
    return np.asarray(d, dtype=np.float64)[:, None] * _dense(b)


# ---------------------------------------------------------------------------
# GCN — reference gnncompose/gcn.py
# ---------------------------------------------------------------------------

PRECOMPUTE, DYNAMIC = "precompute", "dynamic"
AGGREGATE_FIRST, UPDATE_FIRST = "aggregate_first", "update_first"


def ordering_heuristic(k1: int, k2: int) -> str:
    """reference gcn.py:47-55: update first iff k2 < k1."""
    if k1 < 1 or k2 < 1:
        raise ValueError("embedding sizes must be >= 1")
    return UPDATE_FIRST if k2 < k1 else AGGREGATE_FIRST


def precompute_normalized(a_tilde: Csr, d: np.ndarray) -> Csr:
    """reference gcn.py:103-112: Ñ as a k=1 SDDMM with b = c = d[:, None]."""
    dc = np.asarray(d, dtype=np.float64)[:, None]
    return sddmm(a_tilde, dc, dc)


def _aggregate_update(agg, a, h, w, order):
    """reference gcn.py:119-122."""
    if order == UPDATE_FIRST:
        return agg(a, gemm(h, w))
    return gemm(agg(a, h), w)


@dataclass
class GcnGraph:
    """reference gcn.py:76-100 (NormalizedGraph)."""

    a_tilde: Csr
    d_inv_sqrt: np.ndarray
    n_tilde: Csr | None = None

    @classmethod
    def from_adjacency(cls, a: Csr, precompute: bool = True) -> "GcnGraph":
        a_t = add_self_loops(a)
        g = cls(a_t, inv_sqrt_degrees(a_t))
        if precompute:
            g.n_tilde = precompute_normalized(a_t, g.d_inv_sqrt)
        return g


def gcn_layer(g: GcnGraph, h, w, composition: str, order: str | None = None) -> np.ndarray:
    """reference gcn.py:125-161.  ``order=None`` is the reference heuristic;
    a forced order goes through the same _aggregate_update as the reference's
    private gcn.py:119-122."""
    h, w = _dense(h), _dense(w)
    order = order or ordering_heuristic(w.shape[0], w.shape[1])
    if composition == PRECOMPUTE:
        if g.n_tilde is None:
            g.n_tilde = precompute_normalized(g.a_tilde, g.d_inv_sqrt)
        return np.maximum(_aggregate_update(spmm, g.n_tilde, h, w, order), 0.0)
    agg = spmm_unweighted if g.a_tilde.has_unit_values else spmm
    scaled = scale_rows(g.d_inv_sqrt, h)
    out = _aggregate_update(agg, g.a_tilde, scaled, w, order)
    return np.maximum(scale_rows(g.d_inv_sqrt, out), 0.0)


# ---------------------------------------------------------------------------
# GAT — reference gnncompose/gat.py
# ---------------------------------------------------------------------------

REUSE, RECOMPUTE = "reuse", "recompute"


def edge_softmax(a: Csr, s, t, slope: float) -> np.ndarray:
    """reference gat.py:72-95.  ``a`` may be a row-sampled sub-CSR; ``s`` is
    indexed by the local row, ``t`` by the global column."""
    s = np.ascontiguousarray(s, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    out = np.zeros(a.nnz)
    _load().oracle_edge_softmax_f64(a.n_rows, _p64(a.row_ptr), _p64(a.col_idx), _pf(s), _pf(t),
                                    float(slope), _pf(out))
    return out


def atten_calc(a_tilde: Csr, hw, attn_src, attn_dst, slope: float = 0.2) -> Csr:
    """reference gat.py:98-114 (s = hw@a_src, t = hw@a_dst, then edge softmax).

    The "SDDMM over edges" attention variant is the
    same algebra, so this is its oracle too."""
    hw = _dense(hw)
    s = hw @ np.asarray(attn_src, dtype=np.float64).reshape(-1)
    t = hw @ np.asarray(attn_dst, dtype=np.float64).reshape(-1)
    return a_tilde.with_values(edge_softmax(a_tilde, s, t, slope))


def gat_layer(a_tilde: Csr, h, w, attn_src, attn_dst, slope=0.2, composition=REUSE,
              activation="relu") -> np.ndarray:
    """reference gat.py:121-153."""
    h, w = _dense(h), _dense(w)
    hw = gemm(h, w)
    alpha = atten_calc(a_tilde, hw, attn_src, attn_dst, slope)
    if composition == RECOMPUTE:
        out = gemm(spmm(alpha, h), w)
    else:
        out = spmm(alpha, hw)
    return np.maximum(out, 0.0) if activation == "relu" else out


def gat_layer_multihead(a_tilde: Csr, h, w, attn_src, attn_dst, heads: int, slope=0.2,
                        composition=REUSE, activation="relu") -> np.ndarray:
    """SURVEY.md §8(a) A16 (not in the reference): ``heads`` independent
    single-head reference layers on W[:, i*k2:(i+1)*k2], a_src[i], a_dst[i],
    concatenated along columns."""
    w = _dense(w)
    k2 = w.shape[1] // heads
    a_s = np.asarray(attn_src, dtype=np.float64).reshape(heads, k2)
    a_d = np.asarray(attn_dst, dtype=np.float64).reshape(heads, k2)
    outs = [gat_layer(a_tilde, h, w[:, i * k2:(i + 1) * k2], a_s[i], a_d[i], slope,
                      composition, activation) for i in range(heads)]
    return np.concatenate(outs, axis=1)


# ---------------------------------------------------------------------------
# features — reference gnncompose/features.py:49-82
# ---------------------------------------------------------------------------

FEATURE_NAMES = ("n_rows", "n_nnzs", "nnz_den", "nnz_mean", "d_min", "d_max", "d_dentr", "e_dentr")


def extract_features(a: Csr) -> dict:
    n, nnz = a.n_rows, a.nnz
    deg = a.degrees()
    distinct, counts = np.unique(deg, return_counts=True)
    if distinct.size > 1:
        p = counts / n
        d_dentr = float(-(p * np.log(p)).sum() / np.log(distinct.size))
    else:
        d_dentr = 0.0
    if n > 1:
        share = deg[deg > 0] / nnz
        e_dentr = float(-(share * np.log(share)).sum() / np.log(n))
    else:
        e_dentr = 0.0
    return dict(n_rows=n, n_nnzs=nnz, nnz_den=nnz / (n * n), nnz_mean=nnz / n,
                d_min=int(deg.min()), d_max=int(deg.max()), d_dentr=d_dentr, e_dentr=e_dentr)


# ---------------------------------------------------------------------------
# input recipe — reference gnncompose/profiling.py:127-130, 251-259
# ---------------------------------------------------------------------------


def config_rng(seed: int, graph_id: str, k1: int, k2: int) -> np.random.Generator:
    return np.random.default_rng([seed, zlib.crc32(graph_id.encode()), k1, k2])


def draw_inputs(rng, n, k1, k2, model="gcn"):
    h = rng.uniform(-0.5, 0.5, size=(n, k1))
    w = rng.uniform(-0.5, 0.5, size=(k1, k2))
    out = {"h": h, "w": w}
    if model == "gat":
        out["attn_src"] = rng.uniform(-0.5, 0.5, size=k2)
        out["attn_dst"] = rng.uniform(-0.5, 0.5, size=k2)
    return out


# ---------------------------------------------------------------------------
# row partition — SURVEY.md §8(a) A18 (not in the reference)
# ---------------------------------------------------------------------------


def partition_rows(row_ptr, parts: int) -> np.ndarray:
    """nnz-balanced contiguous row blocks: bounds[p] = searchsorted(row_ptr,
    ceil(p*m/P), 'left') for 0<p<P, bounds[0]=0, bounds[P]=n."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = row_ptr.size - 1
    m = int(row_ptr[-1])
    b = np.empty(parts + 1, dtype=np.int64)
    b[0], b[parts] = 0, n
    for p in range(1, parts):
        target = -(-p * m // parts)
        b[p] = min(int(np.searchsorted(row_ptr, target, side="left")), n)
    return b


# ---------------------------------------------------------------------------
# comparison metric — reference tests/helpers.py:68-72
# ---------------------------------------------------------------------------


def rel_err(actual, expected) -> float:
    """max|a-e| / max(1, max|e|) — the reference's normwise metric."""
    actual = np.asarray(actual, dtype=np.float64)
    expected = np.asarray(expected, dtype=np.float64)
    scale = max(1.0, float(np.abs(expected).max()) if expected.size else 1.0)
    if actual.size == 0:
        return 0.0
    return float(np.abs(actual - expected).max()) / scale
