"""Hybrid aggregation for power-law graphs: the dense hub block on the tensor
cores, the sparse tail on the SpMM kernel.

On a dense power-law graph (Reddit-shaped: mean degree ~490) the SpMM is
bound by L2 bandwidth, not HBM: every edge gathers a K-wide row of X and the
most-referenced columns are gathered again and again.  Splitting the columns
into the T most-referenced ("hub") columns and the rest turns the hub part of

    C = D Ã D X          (the reference's dynamic form, gcn.py:137-155;
                          precompute's Ñ = D Ã D, gcn.py:103-112)

into a dense product whose operand tiles are reused from shared memory:

    C_hub = D · A_hub · (D X)[hub_cols],   A_hub ∈ {0,1}^{n × T}

computed by ``gc_hub_gemm_bf16x3`` (tcgen05 kind::f16): A_hub is exact in
bf16 and (D X)[hub_cols] is split into three bf16 terms that together carry
its fp32 mantissa, so the hub part keeps fp32 precision.  The tail SpMM then
accumulates the remaining columns on top (GC_ACCUMULATE).  Only the
summation order differs from the plain SpMM.

The split applies to a unit-valued Ã (the reference's own generated graphs and
``has_unit_values`` case); T is chosen per (pattern, K) by timing the
candidates once, like the SpMM variant autotuner (reference tiling.py:311-364
is the CPU analogue).  "0" in GNNC_HUB_SPLIT disables it; a number forces T.
"""

from __future__ import annotations

import os

import torch

from . import _native as nat
from .sparse import CsrMatrix, ShapeError, _ld, _require_cuda, _spmm, _stream, _timed_call

HUB_SPLIT = os.environ.get("GNNC_HUB_SPLIT", "auto")  # auto | 0 | <T>
HUB_T_CANDIDATES = (1024, 2048, 4096, 8192)
HUB_MIN_NNZ = 1 << 24            # smaller graphs stay on the SpMM alone
HUB_MIN_DENSITY = 0.02           # mean density of the hub block worth a dense product
HUB_MEM_BUDGET = 8 << 30         # bytes of A_hub per pattern


class HubPlan:
    """Column split of one pattern: hub columns, the dense 0/1 hub block
    (bf16, row-major n × T) and the tail pattern (CSR without the hub
    columns; ``keep`` maps tail positions back to the full pattern)."""

    def __init__(self, a: CsrMatrix, T: int):
        if T % 64 or T <= 0 or T > a.n_cols:
            raise ShapeError(f"hub split: T={T} must be a positive multiple of 64 <= n_cols")
        dev = a.device
        counts = torch.bincount(a.col_idx.long(), minlength=a.n_cols)
        hub = torch.topk(counts, T).indices.sort().values
        pos = torch.full((a.n_cols,), -1, dtype=torch.int64, device=dev)
        pos[hub] = torch.arange(T, device=dev)
        colpos = pos[a.col_idx.long()]
        is_hub = colpos >= 0
        rows = a.row_of_nnz()
        self.T = T
        self.hub_cols = hub.to(torch.int32).contiguous()
        self.a_hub = torch.zeros(a.n_rows, T, dtype=torch.bfloat16, device=dev)
        self.a_hub[rows[is_hub], colpos[is_hub]] = 1.0
        keep = torch.nonzero(~is_hub).flatten()
        cnt = torch.bincount(rows[keep], minlength=a.n_rows)
        rp = torch.zeros(a.n_rows + 1, dtype=torch.int32, device=dev)
        rp[1:] = torch.cumsum(cnt, 0).to(torch.int32)
        self.keep = keep
        self.hub_edges = int(is_hub.sum())
        self.tail = CsrMatrix(a.n_rows, a.n_cols, rp, a.col_idx[keep].contiguous(),
                              torch.ones(keep.numel(), dtype=torch.float32, device=dev),
                              validate=False, device=dev)
        self.tail._unit = True
        self._tail_vals: dict = {}

    def tail_block(self, values: torch.Tensor | None, lo: int, hi: int) -> CsrMatrix:
        """Rows [lo, hi) of the tail pattern, carrying ``values`` (a
        same-pattern matrix's values, e.g. Ñ's, gathered at the tail positions)
        or unit values; cached per (values tensor, row range)."""
        vkey = None if values is None else (values.data_ptr(), values._version)
        if vkey not in self._tail_vals:
            self._tail_vals = {k: v for k, v in self._tail_vals.items() if k is None}
            self._tail_vals[vkey] = ({}, self.tail if values is None
                                     else self.tail.with_values(values[self.keep].contiguous()))
        blocks, full = self._tail_vals[vkey]
        if (lo, hi) == (0, full.n_rows):
            return full
        if (lo, hi) not in blocks:
            blocks[(lo, hi)] = full.take_rows(lo, hi)
            blocks[(lo, hi)]._unit = values is None
        return blocks[(lo, hi)]


def hub_plan(a: CsrMatrix, T: int) -> HubPlan:
    key = ("hubsplit", int(T))
    if key not in a._plans:
        a._plans[key] = HubPlan(a, T)
    return a._plans[key]


def pack(a: CsrMatrix, x: torch.Tensor, d: torch.Tensor, T: int) -> torch.Tensor:
    """The hub operand (D X)[hub_cols] as three bf16 terms, K-major."""
    plan = hub_plan(a, T)
    lib = nat.load()
    K = x.shape[1]
    kp = int(lib.gc_hub_terms_rows(K))
    bt = torch.empty(3 * kp * T, dtype=torch.bfloat16, device=x.device)
    nat.check(lib.gc_hub_pack_bf16x3(x.data_ptr(), _ld(x), K, plan.hub_cols.data_ptr(), T,
                                     d.data_ptr(), bt.data_ptr(), _stream(x.device)), "hub_pack")
    return bt


def hybrid_aggregate(a: CsrMatrix, x: torch.Tensor, d: torch.Tensor, T: int, *,
                     d_row: torch.Tensor | None = None, values: torch.Tensor | None = None,
                     relu: bool = False, out: torch.Tensor | None = None,
                     accumulate: bool = False, rows: tuple[int, int] | None = None,
                     packed: torch.Tensor | None = None) -> torch.Tensor:
    """C = epi(D_row Ã D X) for a unit-valued pattern ``a`` via the hub split
    (``d`` scales the columns; ``d_row`` the rows, default ``d`` itself for a
    square pattern).  ``values`` (optional) are a same-pattern matrix's values
    used for the tail instead of d_i·d_j (the precompute composition streams
    Ñ's values).  ``accumulate``: C += ... (ReLU on the total).  ``rows=(lo,
    hi)`` computes that row block only (``out`` then has hi-lo rows);
    ``packed`` reuses one ``pack`` across row blocks."""
    dev = _require_cuda(a.col_idx, x, d)
    if x.dim() != 2 or x.shape[0] != a.n_cols or x.stride(1) != 1:
        raise ShapeError("hybrid_aggregate: x must be a row-major n_cols x K tensor")
    if d_row is None:
        if a.n_rows != a.n_cols:
            raise ShapeError("hybrid_aggregate: d_row is required for a rectangular pattern")
        d_row = d
    K = x.shape[1]
    lo, hi = rows if rows is not None else (0, a.n_rows)
    plan = hub_plan(a, T)
    if out is None:
        if accumulate:
            raise ValueError("hybrid_aggregate: accumulate needs an output")
        out = torch.empty(hi - lo, K, dtype=torch.float32, device=dev)
    elif tuple(out.shape) != (hi - lo, K) or out.stride(1) != 1:
        raise ShapeError(f"hybrid_aggregate: out must be a row-major {hi - lo}x{K} tensor")
    lib = nat.load()
    st = _stream(dev)
    tail = plan.tail_block(values, lo, hi)
    a_hub = plan.a_hub[lo:hi]
    dr = d_row[lo:hi]
    flags = nat.GC_ACCUMULATE if accumulate else 0

    def run():
        bt = packed if packed is not None else pack(a, x, d, T)
        nat.check(_timed_call("hub_gemm", dev, lambda: lib.gc_hub_gemm_bf16x3(
            a_hub.data_ptr(), T, hi - lo, T, bt.data_ptr(), K, out.data_ptr(), _ld(out),
            dr.data_ptr(), flags, st)), "hub_gemm")
        if values is None:
            _spmm(tail, x, weighted=False, d_row=dr, d_col=d, relu=relu, out=out,
                  accumulate=True, timer="spmm_tail")
        else:
            _spmm(tail, x, weighted=True, relu=relu, out=out, accumulate=True, timer="spmm_tail")
        return 0

    _timed_call("spmm", dev, run)
    return out


def _candidates(a: CsrMatrix) -> list[int]:
    counts = torch.bincount(a.col_idx.long(), minlength=a.n_cols)
    top = torch.sort(counts, descending=True).values.double().cumsum(0)
    out = []
    for T in HUB_T_CANDIDATES:
        if T > a.n_cols // 8 or a.n_rows * T * 2 > HUB_MEM_BUDGET:
            continue
        if float(top[T - 1]) / (a.n_rows * T) >= HUB_MIN_DENSITY:
            out.append(T)
    return out


def choose_split(a: CsrMatrix, x: torch.Tensor, d: torch.Tensor, *,
                 d_row: torch.Tensor | None = None, values: torch.Tensor | None = None) -> int:
    """T for (pattern, K): 0 (plain SpMM) unless a hub split is measurably
    faster.  Every candidate is timed once (median of 3 after a warm launch)
    on the first call and the choice is cached on the pattern."""
    mode = str(HUB_SPLIT)
    if mode == "0" or not a.has_unit_values:
        return 0
    if d_row is None:
        if a.n_rows != a.n_cols:
            return 0
        d_row = d
    if mode != "auto":
        return int(mode)
    K = x.shape[1]
    key = ("hubsplit-choice", int(K), values is not None)
    if key in a._plans:
        return a._plans[key]
    if a.nnz < HUB_MIN_NNZ or x.stride(1) != 1:
        a._plans[key] = 0
        return 0
    cands = _candidates(a)
    if not cands:
        a._plans[key] = 0
        return 0
    scratch = torch.empty(a.n_rows, K, dtype=torch.float32, device=x.device)
    src = a if values is None else a.with_values(values)

    def plain():
        _spmm(src, x, weighted=values is not None, d_row=None if values is not None else d_row,
              d_col=None if values is not None else d, out=scratch, timer=None)

    def timed(fn) -> float:
        fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(3)]
        for e0, e1 in ev:
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        return sorted(e0.elapsed_time(e1) for e0, e1 in ev)[1]

    times = {0: timed(plain)}
    for T in cands:
        times[T] = timed(lambda T=T: hybrid_aggregate(a, x, d, T, d_row=d_row, values=values,
                                                      out=scratch))
    best = min(times, key=times.get)
    if best and times[best] >= 0.97 * times[0]:
        best = 0
    for T in cands:  # keep only the chosen block resident
        if T != best:
            a._plans.pop(("hubsplit", T), None)
    a._plans[key] = best
    a._plans[key + ("times",)] = {str(T): round(t, 4) for T, t in times.items()}
    return best
