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

On the layer path (``gat_layer*``) the reassociated form never materialises
α: one kernel computes the edge softmax online inside the aggregation
(SURVEY.md §8(f) N1).  The recompute composition also skips HW entirely:
s = H (W a_src), t = H (W a_dst) needs only two k1-vectors (gat.py:140 forms
HW just for the scores).

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
from .sparse import (
    CsrMatrix,
    gat_sddmm_aggregate,
    ShapeError,
    _Operand,
    _ld,
    _require_cuda,
    _stream,
    call_spmm_hook,
    gat_aggregate,
    gemm,
    gemm_f16rows,
    get_gemm_precision,
    pack_rows_f16,
    relu_,
    spmm,
)

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
    heavy = a_tilde.softmax_heavy_rows()
    if spec.attention is AttentionForm.SDDMM:
        s_work = torch.empty(H, n, dtype=torch.float32, device=dev)
        rc = lib.gc_attn_sddmm_f32(a_tilde.row_ptr.data_ptr(), a_tilde.col_idx.data_ptr(),
                                   hwt.data_ptr(), _ld(hwt), None, 0, k2, H, a_src.data_ptr(),
                                   a_dst.data_ptr(), float(spec.leaky_slope), n, m,
                                   heavy.data_ptr(), heavy.numel(), s_work.data_ptr(),
                                   alpha.data_ptr(), st)
        nat.check(rc, "attn_sddmm")
    else:
        s = torch.empty(H, n, dtype=torch.float32, device=dev)
        t = torch.empty(H, n, dtype=torch.float32, device=dev)
        nat.check(lib.gc_node_proj_f32(hwt.data_ptr(), _ld(hwt), n, k2, H, k2, a_src.data_ptr(),
                                       a_dst.data_ptr(), s.data_ptr(), t.data_ptr(), st), "node_proj")
        nat.check(lib.gc_edge_softmax_f32(a_tilde.row_ptr.data_ptr(), a_tilde.col_idx.data_ptr(),
                                          s.data_ptr(), t.data_ptr(), H, float(spec.leaky_slope), n, m,
                                          heavy.data_ptr(), heavy.numel(), alpha.data_ptr(), st),
                  "edge_softmax")
    return AttentionMatrix(alpha=a_tilde.with_values(alpha[0]), values=alpha if H > 1 else None)


def _projections(x: torch.Tensor, spec: GatLayerSpec, a_src: torch.Tensor, a_dst: torch.Tensor,
                 width: int, head_stride: int) -> tuple[torch.Tensor, torch.Tensor]:
    """s[h], t[h] = X[:, h-block] · a_src[h], · a_dst[h] for every head."""
    dev = x.device
    n, H = x.shape[0], spec.heads
    s = torch.empty(H, n, dtype=torch.float32, device=dev)
    t = torch.empty(H, n, dtype=torch.float32, device=dev)
    nat.check(nat.load().gc_node_proj_f32(x.data_ptr(), _ld(x), n, width, H, head_stride,
                                          a_src.data_ptr(), a_dst.data_ptr(), s.data_ptr(),
                                          t.data_ptr(), _stream(dev)), "node_proj")
    return s, t


def _folded_attention_vectors(spec: GatLayerSpec) -> tuple[torch.Tensor, torch.Tensor]:
    """u_h = W_h a_src_h, v_h = W_h a_dst_h (k1-vectors, heads concatenated),
    cached on the spec; exact-fp32 GEMVs through the library."""
    w = spec.weights
    key = (w.data_ptr(), w._version, spec.attn_src.data_ptr(), spec.attn_src._version,
           spec.attn_dst.data_ptr(), spec.attn_dst._version)
    cache = getattr(spec, "_uv_cache", None)
    if cache is not None and cache[0] == key:
        return cache[1], cache[2]
    k1, k2, H = spec.k1, spec.k2, spec.heads
    u = torch.empty(H * k1, dtype=torch.float32, device=w.device)
    v = torch.empty(H * k1, dtype=torch.float32, device=w.device)
    for i in range(H):
        wi = w[:, i * k2:(i + 1) * k2]
        ab = torch.stack([spec.attn_src[i * k2:(i + 1) * k2], spec.attn_dst[i * k2:(i + 1) * k2]], 1)
        uv = gemm(wi, ab.contiguous(), precision="fp32")
        u[i * k1:(i + 1) * k1] = uv[:, 0]
        v[i * k1:(i + 1) * k1] = uv[:, 1]
    spec._uv_cache = (key, u, v)
    return u, v


def _check_h(a_tilde: CsrMatrix, h, spec: GatLayerSpec) -> None:
    shape = tuple(h.shape)
    if len(shape) != 2 or shape != (a_tilde.n_rows, spec.k1):
        raise ShapeError(f"embeddings shape {shape} != ({a_tilde.n_rows}, {spec.k1})")


def _reuse_f16rows(a_tilde: CsrMatrix, x: torch.Tensor, spec: GatLayerSpec) -> bool:
    """TF32 class, several heads, reassociated attention, each head's HW at
    most 256 wide or a multiple of 256 (one scale per 256-column chunk) and
    large enough for fp16 gathers: each head's GEMM emits
    its fp16 rows directly (no fp32 HW written and re-read by the packs) —
    arxiv 4 heads K = 256 1.11 vs 1.17 ms; one head keeps the single GEMM +
    pack with fused scores (0.310 vs 0.315 ms), profiles/data/gat_reuse_f16_r02.json."""
    from . import gcn

    k2 = spec.k2
    return (spec.heads > 1 and spec.attention is AttentionForm.REASSOC
            and a_tilde.n_rows == a_tilde.n_cols
            and gcn.HALF_GATHER and get_gemm_precision() == "tf32" and x.is_cuda
            and k2 % 8 == 0 and (k2 <= 256 or k2 % 256 == 0)
            and x.shape[0] * k2 * 4 > gcn.HALF_MIN_BYTES)


def _reuse_reassoc_f16rows(a_tilde: CsrMatrix, x: torch.Tensor, spec: GatLayerSpec,
                           relu: bool) -> torch.Tensor:
    """Reuse composition, reassociated attention, TF32 class: per head,
    HW_h as fp16 rows straight from the GEMM epilogue (gemm_f16rows); the
    node scores s = H (W_h a_src), t = H (W_h a_dst) from the folded vectors
    in one pass over H for every head (the recompute path's projections —
    the same values up to fp32 association)."""
    k1, k2, H = spec.k1, spec.k2, spec.heads
    u, v = _folded_attention_vectors(spec)
    s, t = _projections(x, spec, u, v, k1, 0)
    out = torch.empty(a_tilde.n_rows, k2 * H, dtype=torch.float32, device=x.device)
    for i in range(H):
        cs = slice(i * k2, (i + 1) * k2)
        hr = gemm_f16rows(x, spec.weights[:, cs].contiguous())
        if hr is None:  # outside the fused epilogue's range: fp32 GEMM, then pack
            hr = pack_rows_f16(gemm(x, spec.weights[:, cs].contiguous()))
        gat_aggregate(a_tilde, s[i], t[i], spec.leaky_slope, hr, relu=relu, out=out[:, cs])
    return out


def gat_layer_reuse(a_tilde: CsrMatrix, h, spec: GatLayerSpec, *, spmm_fn=None):
    """HW once, reused for attention and aggregation (SpMM at k2) — gat.py:121-129."""
    _check_h(a_tilde, h, spec)
    op = _Operand(h, a_tilde.device)
    relu = spec.activation == "relu"
    if spmm_fn is None and _reuse_f16rows(a_tilde, op.t, spec):
        return op.wrap(_reuse_reassoc_f16rows(a_tilde, op.t, spec, relu))
    hw = gemm(op.t, spec.weights)
    k2, H = spec.k2, spec.heads
    if spmm_fn is not None:
        att = atten_calc(a_tilde, hw, spec)
        outs = [call_spmm_hook(spmm_fn, att.head(i), hw[:, i * k2:(i + 1) * k2].contiguous())
                for i in range(H)]
        out = torch.cat(outs, 1).contiguous()
        return op.wrap(relu_(out) if relu else out)
    out = torch.empty(a_tilde.n_rows, k2 * H, dtype=torch.float32, device=hw.device)
    half = _half(hw[:, :k2])
    if spec.attention is AttentionForm.SDDMM:
        if a_tilde.n_rows == a_tilde.n_cols:
            # fused: the gathered HW_j row gives its score and its aggregated term.
            # fp32 rows even in the TF32 class: the score operands double the
            # live registers of this mode, and with fp16 rows its occupancy
            # halves (arxiv K = 256: 0.67 vs 0.43 ms; ncu 22 % warps active,
            # profiles/r02_ncu_summary.md); gc_gat_sddmm_aggregate_f32 accepts
            # fp16 rows (GC_SPMM_B_F16) for callers that want the bytes
            a_src, a_dst = spec.attn_src.to(hw.device), spec.attn_dst.to(hw.device)
            done = all(gat_sddmm_aggregate(a_tilde, a_src[i * k2:(i + 1) * k2],
                                           a_dst[i * k2:(i + 1) * k2], spec.leaky_slope,
                                           hw[:, i * k2:(i + 1) * k2], relu=relu,
                                           out=out[:, i * k2:(i + 1) * k2])
                       is not None for i in range(H))
            if done:
                return op.wrap(out)
        att = atten_calc(a_tilde, hw, spec)
        for i in range(H):
            spmm(att.head(i), hw[:, i * k2:(i + 1) * k2], relu=relu, out=out[:, i * k2:(i + 1) * k2])
        return op.wrap(out)
    if a_tilde.n_rows != a_tilde.n_cols:
        raise ShapeError("attention expects a square adjacency")
    a_src, a_dst = spec.attn_src.to(hw.device), spec.attn_dst.to(hw.device)
    if half and k2 % 4 == 0:
        # TF32 class: each head's slice of HW is packed to fp16 rows and its
        # node scores s, t come out of the same pass (rows read once)
        for i in range(H):
            cs = slice(i * k2, (i + 1) * k2)
            hr, st = pack_rows_f16(hw[:, cs], proj=torch.stack([a_src[cs], a_dst[cs]]))
            gat_aggregate(a_tilde, st[0], st[1], spec.leaky_slope, hr, relu=relu, out=out[:, cs])
        return op.wrap(out)
    s, t = _projections(hw, spec, a_src, a_dst, k2, k2)
    for i in range(H):
        b = hw[:, i * k2:(i + 1) * k2]
        gat_aggregate(a_tilde, s[i], t[i], spec.leaky_slope, pack_rows_f16(b) if half else b,
                      relu=relu, out=out[:, i * k2:(i + 1) * k2])
    return op.wrap(out)


def gat_layer_recompute(a_tilde: CsrMatrix, h, spec: GatLayerSpec, *, spmm_fn=None):
    """Aggregate the raw H (SpMM at k1) then update with one more GEMM —
    gat.py:132-145.  In the reassociated form the scores come from H and the
    folded vectors W a (no HW GEMM); the "sddmm" form needs HW for its
    per-edge dot products, as the reference's recompute does."""
    _check_h(a_tilde, h, spec)
    op = _Operand(h, a_tilde.device)
    relu = spec.activation == "relu"
    k1, k2, H = spec.k1, spec.k2, spec.heads
    dev = op.t.device
    out = torch.empty(a_tilde.n_rows, k2 * H, dtype=torch.float32, device=dev)
    if spmm_fn is not None or spec.attention is AttentionForm.SDDMM:
        hw = gemm(op.t, spec.weights)
        att = atten_calc(a_tilde, hw, spec)
        agg = spmm_fn if spmm_fn is not None else spmm
        for i in range(H):
            ah = call_spmm_hook(agg, att.head(i), op.t)
            gemm(ah, spec.weights[:, i * k2:(i + 1) * k2], relu=relu, out=out[:, i * k2:(i + 1) * k2])
        return op.wrap(out)
    if a_tilde.n_rows != a_tilde.n_cols:
        raise ShapeError("attention expects a square adjacency")
    u, v = _folded_attention_vectors(spec)
    if _half(op.t) and k1 % 4 == 0 and 2 * H <= 16:
        # one pack of H shared by the heads, with every head's s, t from the
        # same pass over the rows
        x, st = pack_rows_f16(op.t, proj=torch.cat([u.view(H, k1), v.view(H, k1)]))
        s, t = st[:H], st[H:]
    else:
        s, t = _projections(op.t, spec, u, v, k1, 0)
        x = pack_rows_f16(op.t) if _half(op.t) else op.t  # one pack, shared by the heads
    for i in range(H):
        ah = gat_aggregate(a_tilde, s[i], t[i], spec.leaky_slope, x)
        gemm(ah, spec.weights[:, i * k2:(i + 1) * k2], relu=relu, out=out[:, i * k2:(i + 1) * k2])
    return op.wrap(out)


def _half(x: torch.Tensor) -> bool:
    """TF32 class: the aggregation gathers fp16 rows of its operand (as the
    GCN layers do, gcn.half_gather)."""
    from .gcn import half_gather

    return half_gather(x)


def gat_layer(a_tilde: CsrMatrix, h, spec: GatLayerSpec, *, spmm_fn=None):
    if spec.composition is GatComposition.RECOMPUTE:
        return gat_layer_recompute(a_tilde, h, spec, spmm_fn=spmm_fn)
    return gat_layer_reuse(a_tilde, h, spec, spmm_fn=spmm_fn)
