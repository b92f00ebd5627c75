"""Row-sampled oracle layers for the full BASELINE shapes (SURVEY.md §8(c)
step 5).  TEST INFRASTRUCTURE: the checker only (used by tests/ and by
bench.py's parity checks; never by the product package).

The layer output rows ``rows`` depend on the operand rows of their
neighbours only, so the reference layer (gcn.py:125-161, gat.py:121-153) is
evaluated on the sub-CSR of those rows with its columns remapped onto the
union of neighbours (``needed``): the GEMMs and GEMVs run on ``needed`` rows
instead of all n, with the reference kernels' arithmetic (oracle C kernels,
float64, same accumulation order).  Graph prep (Ã, D^-1/2) comes from the
oracle's own restatement of the reference, not from the device.
"""

from __future__ import annotations

import numpy as np

from . import gnn_oracle as orc


def _remap(sub: "orc.Csr", rows: np.ndarray):
    """(sub-CSR with columns in ``needed`` index space, needed ids)."""
    needed = np.unique(np.concatenate([sub.col_idx, rows]))
    cols = np.searchsorted(needed, sub.col_idx)
    return orc.Csr(sub.n_rows, needed.size, sub.row_ptr, cols, sub.values), needed


def needed_rows(at: "orc.Csr", rows: np.ndarray) -> np.ndarray:
    """The operand rows the outputs ``rows`` depend on."""
    return _remap(at.take_rows(np.asarray(rows, dtype=np.int64)), rows)[1]


def _rows_of(h, needed):
    return np.ascontiguousarray(h(needed) if callable(h) else h[needed], dtype=np.float64)


def gcn_rows(at: "orc.Csr", d: np.ndarray, h, w: np.ndarray, rows: np.ndarray,
             composition: str, order: str) -> np.ndarray:
    """Reference GCN layer output restricted to ``rows`` (float64).  ``h``:
    the n x k1 operand, or a callable returning its rows for an index array."""
    rows = np.asarray(rows, dtype=np.int64)
    sub, needed = _remap(at.take_rows(rows), rows)
    hn = _rows_of(h, needed)
    w = np.asarray(w, dtype=np.float64)
    if composition == "precompute":
        # Ñ = sddmm(Ã, d, d): a_ij * (d_i * d_j)  (gcn.py:103-112, sparse.py:222-232)
        ri = np.repeat(rows, np.diff(sub.row_ptr))
        nt = sub.with_values(sub.values * (d[ri] * d[needed[sub.col_idx]]))
        out = orc.spmm(nt, orc.gemm(hn, w)) if order == "update_first" else \
            orc.gemm(orc.spmm(nt, hn), w)
        return np.maximum(out, 0.0)
    agg = orc.spmm_unweighted if at.has_unit_values else orc.spmm
    scaled = orc.scale_rows(d[needed], hn)
    out = agg(sub, orc.gemm(scaled, w)) if order == "update_first" else \
        orc.gemm(agg(sub, scaled), w)
    return np.maximum(orc.scale_rows(d[rows], out), 0.0)


def gat_rows(at: "orc.Csr", h, w: np.ndarray, a_src: np.ndarray, a_dst: np.ndarray,
             heads: int, rows: np.ndarray, composition: str, slope: float = 0.2,
             activation: str = "relu") -> np.ndarray:
    """Reference (multi-head = per-head concatenation) GAT layer output on
    ``rows``: HW, s = HW a_src, t = HW a_dst, edge softmax, aggregation.
    ``h`` as in :func:`gcn_rows`."""
    rows = np.asarray(rows, dtype=np.int64)
    sub, needed = _remap(at.take_rows(rows), rows)
    hn = _rows_of(h, needed)
    w = np.asarray(w, dtype=np.float64)
    k2 = w.shape[1] // heads
    pos = np.searchsorted(needed, rows)
    a_s = np.asarray(a_src, dtype=np.float64).reshape(heads, k2)
    a_d = np.asarray(a_dst, dtype=np.float64).reshape(heads, k2)
    outs = []
    for i in range(heads):
        wi = np.ascontiguousarray(w[:, i * k2:(i + 1) * k2])
        hw = orc.gemm(hn, wi)
        s = hw[pos] @ a_s[i]
        t = hw @ a_d[i]
        alpha = sub.with_values(orc.edge_softmax(sub, s, t, slope))
        out = orc.gemm(orc.spmm(alpha, hn), wi) if composition == "recompute" else orc.spmm(alpha, hw)
        outs.append(np.maximum(out, 0.0) if activation == "relu" else out)
    return np.concatenate(outs, axis=1)


def sample_rows(n: int, count: int, seed: int, heavy: np.ndarray | None = None) -> np.ndarray:
    """``count`` uniformly drawn rows plus (optionally) the given heavy rows."""
    rng = np.random.default_rng(seed)
    r = rng.choice(n, size=min(count, n), replace=False)
    if heavy is not None:
        r = np.concatenate([r, heavy])
    return np.unique(r)
