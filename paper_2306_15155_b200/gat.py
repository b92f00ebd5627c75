"""GAT layer under the reuse and recompute compositions, single- or multi-head.

Drop-in mirror of ``gnncompose/gat.py``.  Both compositions compute HW = H W
once (tcgen05 GEMM) and the edge attention α on the pattern of Ã; they differ
in what is aggregated:

* reuse: α · HW (SpMM at width k2);
* recompute: (α · H) · W (SpMM at width k1, one more GEMM).

The attention itself has two B200 forms (``GatLayerSpec.attention``):

* "reassoc" (the reference's form, gat.py:110-114): per-node projections
  s = HW a_src, t = HW a_dst, then one fused LeakyReLU + edge-softmax kernel
  that gathers only t_j per edge;
* "sddmm": the score of every edge as a k2-wide SDDMM over HW rows
  (a_src·HW_i + a_dst·HW_j), fused with the same LeakyReLU + softmax.

Multi-head (``heads`` > 1, not in the reference): W is
k1 x (heads*k2) and attn vectors have heads*k2 entries; head h uses the column
block h, and outputs are concatenated — identical to ``heads`` independent
single-head layers.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as nat
from .sparse import CsrMatrix, ShapeError, _Operand, _ld, _require_cuda, _stream, gemm, relu_, spmm


class GatComposition(str, Enum):
    REUSE = "reuse"
    RECOMPUTE = "recompute"


class AttentionForm(str, Enum):
    REASSOC = "reassoc"
    SDDMM = "sddmm"


def _vec(x, n: int, device) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float64))
    t = t.reshape(-1)
    if t.numel() != n:
        raise ShapeError("attention vectors must have length k2 (per head)")
    return t.to(device, torch.float32).contiguous()


@dataclass
class GatLayerSpec:
    """Reference gat.py:30-57, plus ``heads`` and ``attention`` extensions."""

    k1: int
    k2: int
    weights: object
    attn_src: object
    attn_dst: object
    leaky_slope: float = 0.2
    composition: GatComposition = GatComposition.REUSE
    activation: str = "relu"  # "relu" or "none"
    heads: int = 1
    attention: AttentionForm = AttentionForm.REASSOC

    def __post_init__(self):
        from .sparse import default_device

        if self.k1 < 1 or self.k2 < 1:
            raise ValueError("embedding sizes must be >= 1")
        if not 1 <= int(self.heads) <= 8:
            raise ValueError("heads must be in [1, 8]")
        self.heads = int(self.heads)
        w = self.weights
        t = w if isinstance(w, torch.Tensor) else torch.from_numpy(np.asarray(w, dtype=np.float64))
        if tuple(t.shape) != (self.k1, self.k2 * self.heads):
            raise ShapeError(f"weights shape {tuple(t.shape)} != ({self.k1}, {self.k2 * self.heads})")
        dev = t.device if t.is_cuda else default_device()
        self.weights = t.to(dev, torch.float32).contiguous()
        self.attn_src = _vec(self.attn_src, self.k2 * self.heads, dev)
        self.attn_dst = _vec(self.attn_dst, self.k2 * self.heads, dev)
        if not 0.0 < self.leaky_slope < 1.0:
            raise ValueError("leaky_slope must lie in (0, 1)")
        self.composition = GatComposition(self.composition)
        self.attention = AttentionForm(self.attention)
        if self.activation not in ("relu", "none"):
            raise ValueError("activation must be 'relu' or 'none'")


@dataclass
class AttentionMatrix:
    """Post-softmax attention on the pattern of Ã (reference gat.py:60-69).
    ``alpha`` is head 0; ``values`` holds all heads as [heads, nnz]."""

    alpha: CsrMatrix
    values: torch.Tensor | None = None

    @property
    def heads(self) -> int:
        return 1 if self.values is None else self.values.shape[0]

    def head(self, h: int) -> CsrMatrix:
        return self.alpha if h == 0 or self.values is None else self.alpha.with_values(self.values[h])

    def row_sums(self) -> torch.Tensor:
        a = self.alpha
        vals = self.values if self.values is not None else a.values[None]
        rows = a.row_of_nnz()
        out = torch.zeros(vals.shape[0], a.n_rows, dtype=torch.float64, device=a.device)
        out.index_add_(1, rows, vals.double())
        return out[0] if self.values is None else out


def atten_calc(a_tilde: CsrMatrix, hw, spec: GatLayerSpec) -> AttentionMatrix:
    """Edge attention: masked LeakyReLU scores + per-row softmax (gat.py:98-114),
    on the GPU, in the form ``spec.attention`` selects."""
    dev = a_tilde.device
    hwt = _Operand(hw, dev).t
    H, k2 = spec.heads, spec.k2
    if tuple(hwt.shape) != (a_tilde.n_rows, k2 * H):
        raise ShapeError(f"hw shape {tuple(hwt.shape)} != ({a_tilde.n_rows}, {k2 * H})")
    if a_tilde.n_rows != a_tilde.n_cols:
        raise ShapeError("attention expects a square adjacency")
    _require_cuda(a_tilde.col_idx, hwt)
    n, m = a_tilde.n_rows, a_tilde.nnz
    a_src = spec.attn_src.to(dev)
    a_dst = spec.attn_dst.to(dev)
    alpha = torch.empty(H, m, dtype=torch.float32, device=dev)
    lib = nat.load()
    st = _stream(dev)
    if spec.attention is AttentionForm.SDDMM:
        rc = lib.gc_attn_sddmm_f32(a_tilde.row_ptr.data_ptr(), a_tilde.col_idx.data_ptr(),
                                   hwt.data_ptr(), _ld(hwt), k2, H, a_src.data_ptr(),
                                   a_dst.data_ptr(), float(spec.leaky_slope), n, m,
                                   alpha.data_ptr(), st)
        nat.check(rc, "attn_sddmm")
    else:
        s = torch.empty(H, n, dtype=torch.float32, device=dev)
        t = torch.empty(H, n, dtype=torch.float32, device=dev)
        nat.check(lib.gc_node_proj_f32(hwt.data_ptr(), _ld(hwt), n, k2, H, a_src.data_ptr(),
                                       a_dst.data_ptr(), s.data_ptr(), t.data_ptr(), st), "node_proj")
        nat.check(lib.gc_edge_softmax_f32(a_tilde.row_ptr.data_ptr(), a_tilde.col_idx.data_ptr(),
                                          s.data_ptr(), t.data_ptr(), H, float(spec.leaky_slope), n, m,
                                          alpha.data_ptr(), st), "edge_softmax")
    return AttentionMatrix(alpha=a_tilde.with_values(alpha[0]), values=alpha if H > 1 else None)


def _check_h(a_tilde: CsrMatrix, h, spec: GatLayerSpec) -> None:
    shape = tuple(h.shape)
    if len(shape) != 2 or shape != (a_tilde.n_rows, spec.k1):
        raise ShapeError(f"embeddings shape {shape} != ({a_tilde.n_rows}, {spec.k1})")


def gat_layer_reuse(a_tilde: CsrMatrix, h, spec: GatLayerSpec, *, spmm_fn=None):
    """HW once, reused for attention and aggregation (SpMM at k2) — gat.py:121-129."""
    _check_h(a_tilde, h, spec)
    op = _Operand(h, a_tilde.device)
    relu = spec.activation == "relu"
    hw = gemm(op.t, spec.weights)
    att = atten_calc(a_tilde, hw, spec)
    k2 = spec.k2
    if spmm_fn is not None:
        outs = [spmm_fn(att.head(i), hw[:, i * k2:(i + 1) * k2]) for i in range(spec.heads)]
        out = torch.cat([torch.as_tensor(o, device=hw.device).float() for o in outs], 1).contiguous()
        return op.wrap(relu_(out) if relu else out)
    out = torch.empty(a_tilde.n_rows, k2 * spec.heads, dtype=torch.float32, device=hw.device)
    for i in range(spec.heads):
        spmm(att.head(i), hw[:, i * k2:(i + 1) * k2], relu=relu, out=out[:, i * k2:(i + 1) * k2])
    return op.wrap(out)


def gat_layer_recompute(a_tilde: CsrMatrix, h, spec: GatLayerSpec, *, spmm_fn=None):
    """Aggregate the raw H (SpMM at k1) then update with one more GEMM —
    gat.py:132-145.  HW is still computed once for the attention."""
    _check_h(a_tilde, h, spec)
    op = _Operand(h, a_tilde.device)
    relu = spec.activation == "relu"
    hw = gemm(op.t, spec.weights)
    att = atten_calc(a_tilde, hw, spec)
    k2 = spec.k2
    out = torch.empty(a_tilde.n_rows, k2 * spec.heads, dtype=torch.float32, device=hw.device)
    agg = spmm_fn if spmm_fn is not None else spmm
    for i in range(spec.heads):
        ah = agg(att.head(i), op.t)
        ah = ah if isinstance(ah, torch.Tensor) else torch.as_tensor(ah, device=hw.device).float()
        gemm(ah, spec.weights[:, i * k2:(i + 1) * k2], relu=relu, out=out[:, i * k2:(i + 1) * k2])
    return op.wrap(out)


def gat_layer(a_tilde: CsrMatrix, h, spec: GatLayerSpec, *, spmm_fn=None):
    if spec.composition is GatComposition.RECOMPUTE:
        return gat_layer_recompute(a_tilde, h, spec, spmm_fn=spmm_fn)
    return gat_layer_reuse(a_tilde, h, spec, spmm_fn=spmm_fn)
