"""Row-partitioned GCN and GAT layers across GPUs.

One process per GPU (``torch.distributed``, NCCL over NVLink on the box,
gloo in the CPU tests).  Ã is cut into contiguous, nnz-balanced row blocks
(``partition_rows`` — the C-ABI host function, bit-exact with the oracle);
rank p owns rows [b_p, b_{p+1}) with global column ids.  Per layer exactly one
all-gather assembles the operand the local aggregation gathers:

    composition              all-gathered operand (one collective)
    GCN A(HW)                H_p W          (d ⊙ folded into the GEMM epilogue)
    GCN (AH)W                H_p
    GAT reuse, reassoc       [H_p W | t_p]  (gat.py:121-129)
    GAT reuse, sddmm         H_p W          (scores from the gathered rows)
    GAT recompute, reassoc   [H_p | t_p]    (gat.py:132-145; t_p = H_p W a_dst)
    GAT recompute, sddmm     [H_p | H_p W]  (α needs HW rows, the SpMM H rows)

Output rows stay partitioned and feed the next layer.  Blocks are padded to
the largest block for ``all_gather_into_tensor``; the local pattern's column
ids are remapped once into that padded layout (``RowPartition.padded``) so the
gathered buffer is used in place, and the gather buffers are reused across
layers (cached per partition, width and role).

Overlap (``overlap=True``, GCN): the local block of the
pattern is split by column into the edges whose source row this rank owns
(aggregated straight from its own operand block, while the all-gather is in
flight) and the remote edges.  The remote pass accumulates into the local one
(``out += d_i * acc``; ReLU on the total).  (GAT keeps one pass: its online
softmax would need the two passes' (max, sum) states merged.)

Capacity path: :meth:`RowPartition.from_file` reads only this rank's rows of a
``.gcsr`` file of Ã (the row_ptr — O(n) — is read whole to cut the blocks and
to form D^-1/2), so no rank materialises the whole graph.

The compute ops are injectable (``ops``) so the host logic — partition,
padding, gather, remapping, assembly — is testable on CPU with gloo and the
oracle standing in for the CUDA kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat
from .sparse import CsrMatrix, HalfRows, ShapeError, pack_rows_f16


def partition_rows(row_ptr, parts: int) -> np.ndarray:
    """nnz-balanced contiguous row blocks: bounds[p] = first r with
    row_ptr[r] >= ceil(p*nnz/P) (C ABI gc_partition_rows).  A device-resident
    row_ptr is partitioned in place (:func:`partition_rows_device`)."""
    if isinstance(row_ptr, torch.Tensor) and row_ptr.is_cuda:
        return partition_rows_device(row_ptr, parts)
    rp = np.ascontiguousarray(
        row_ptr.cpu().numpy() if isinstance(row_ptr, torch.Tensor) else row_ptr, dtype=np.int64)
    out = np.zeros(parts + 1, dtype=np.int64)
    nat.check(nat.load().gc_partition_rows(rp.ctypes.data, rp.size - 1, int(parts), out.ctypes.data),
              "partition_rows")
    return out


def partition_rows_device(row_ptr: torch.Tensor, parts: int) -> np.ndarray:
    """:func:`partition_rows` computed where ``row_ptr`` lives: one scalar
    read (nnz), P-1 lower-bound searches on the device, P+1 bounds back —
    row_ptr itself never crosses to the host.  Bit-identical to the C ABI
    (``searchsorted(left)`` is ``std::lower_bound``)."""
    if parts < 1:
        raise ValueError("partition_rows: parts must be >= 1")
    n = row_ptr.numel() - 1
    if n < 0:
        raise ValueError("partition_rows: empty row_ptr")
    m = int(row_ptr[-1])
    p = torch.arange(1, parts, dtype=torch.int64)
    target = ((p * m + parts - 1) // parts).to(row_ptr.device, row_ptr.dtype)
    hit = torch.searchsorted(row_ptr.contiguous(), target, right=False).clamp_(max=n)
    out = np.empty(parts + 1, dtype=np.int64)
    out[0], out[parts] = 0, n
    out[1:parts] = hit.cpu().numpy()
    return out


@dataclass
class RowPartition:
    rank: int
    world: int
    bounds: np.ndarray  # P+1 row boundaries
    local: CsrMatrix  # rows [lo, hi) of Ã (or Ñ), global column ids

    @property
    def lo(self) -> int:
        return int(self.bounds[self.rank])

    @property
    def hi(self) -> int:
        return int(self.bounds[self.rank + 1])

    @property
    def rows(self) -> int:
        return self.hi - self.lo

    @property
    def max_rows(self) -> int:
        return max(int(np.diff(self.bounds).max()), 1)

    @classmethod
    def of(cls, a: CsrMatrix, rank: int, world: int) -> "RowPartition":
        b = partition_rows(a.row_ptr, world)
        return cls(rank, world, b, a.take_rows(int(b[rank]), int(b[rank + 1])))

    @classmethod
    def from_file(cls, path, rank: int, world: int, device=None) -> tuple["RowPartition", torch.Tensor]:
        """This rank's block of the ``.gcsr`` file of Ã (self loops included)
        and the FULL D^-1/2 vector, reading only the O(n) row_ptr and this
        rank's rows of col_idx/values: the capacity path, where no rank holds
        the whole graph.  Bounds are bit-identical to :meth:`of`."""
        rp = CsrMatrix.read_row_ptr(path)
        b = partition_rows(rp, world)
        local = CsrMatrix.load(path, device=device, rows=(int(b[rank]), int(b[rank + 1])))
        deg = np.diff(rp).astype(np.float64)
        if deg.size and deg.min() <= 0:
            from .sparse import DegenerateNodeError

            raise DegenerateNodeError("zero-degree row: D^-1/2 undefined")
        d = torch.from_numpy((1.0 / np.sqrt(deg)).astype(np.float32)).to(local.device)
        return cls(rank, world, b, local), d

    def _owner_map(self, col: torch.Tensor):
        bounds = torch.as_tensor(self.bounds, device=col.device)
        owner = torch.searchsorted(bounds[1:], col, right=True)
        return owner, owner * self.max_rows + (col - bounds[owner])

    def padded(self) -> CsrMatrix:
        """The local block with its column ids remapped into the padded
        all-gather layout (column j owned by rank q at q * max_rows + j - b_q),
        n_cols = world * max_rows; cached."""
        if getattr(self, "_padded", None) is None:
            a = self.local
            _, cols = self._owner_map(a.col_idx.long())
            pad = CsrMatrix(a.n_rows, self.world * self.max_rows, a.row_ptr, cols, a.values,
                            validate=False, device=a.device)
            pad._unit = a._unit
            self._padded = pad
        return self._padded

    def pad_vector(self, d: torch.Tensor) -> torch.Tensor:
        """A full per-node vector (e.g. D^-1/2) in the padded layout (zeros in
        the padding); cached per source tensor."""
        key = (id(d), d._version)
        hit = getattr(self, "_dpad", None)
        if hit is None or hit[0] != key or hit[1] is not d:
            out = torch.zeros(self.world * self.max_rows, dtype=d.dtype, device=d.device)
            for p in range(self.world):
                lo, hi = int(self.bounds[p]), int(self.bounds[p + 1])
                out[p * self.max_rows: p * self.max_rows + hi - lo] = d[lo:hi]
            self._dpad = (key, d, out)
        return self._dpad[2]

    def split_local_remote(self) -> tuple[CsrMatrix, CsrMatrix]:
        """(edges from owned rows, columns rebased to the local block;
        remaining edges, columns remapped into the padded gather buffer)."""
        if getattr(self, "_lr", None) is None:
            a = self.local
            col = a.col_idx.long()
            rows = a.row_of_nnz()
            own = (col >= self.lo) & (col < self.hi)
            _, padded = self._owner_map(col)

            def sub(mask, cols, n_cols):
                cnt = torch.bincount(rows[mask], minlength=a.n_rows)
                rp = torch.cat([cnt.new_zeros(1), torch.cumsum(cnt, 0)])
                return CsrMatrix(a.n_rows, n_cols, rp, cols[mask], a.values[mask], validate=False,
                                 device=a.device)

            loc = sub(own, col - self.lo, max(self.rows, 1))
            rem = sub(~own, padded, self.world * self.max_rows)
            loc._unit = rem._unit = a._unit
            self._lr = (loc, rem)
        return self._lr

    def gather_buffers(self, k: int, dtype, device, tag: str = "x"):
        """(send [max_rows, k], recv [world*max_rows, k]) reused across layers
        (stream-ordered: the next gather into a buffer follows the kernels
        that read it on the same stream)."""
        cache = self.__dict__.setdefault("_bufs", {})
        key = (tag, int(k), dtype, str(device))
        if key not in cache:
            cache[key] = (torch.zeros(self.max_rows, k, dtype=dtype, device=device),
                          torch.empty(self.world * self.max_rows, k, dtype=dtype, device=device))
        return cache[key]


def all_gather_padded(x_local: torch.Tensor, part: RowPartition, group=None, async_op=False,
                      tag: str = "x"):
    """Padded all-gather: returns (buffer of world*max_rows rows, work handle).
    The buffers are the partition's cached ones (:meth:`RowPartition.gather_buffers`)."""
    k = x_local.shape[1]
    send, full = part.gather_buffers(k, x_local.dtype, x_local.device, tag)
    if x_local.shape[0] == part.max_rows and x_local.is_contiguous():
        send = x_local
    else:
        send[: x_local.shape[0]].copy_(x_local)
    work = dist.all_gather_into_tensor(full, send, group=group, async_op=async_op)
    return full, work


def all_gather_half(hr: HalfRows, part: RowPartition, group=None, async_op=False):
    """All-gather fp16 rows with their scales in ONE collective (TF32 class:
    half the bytes of the fp32 operand): each row travels as its ldh halves
    followed by 8 halves whose first two hold the float32 scale's bits.
    Returns (HalfRows over the padded gather buffer, work handle, finish) —
    call ``finish()`` after ``work.wait()`` to extract the scales."""
    if hr.chunks != 1:
        raise ShapeError("all_gather_half: one scale per row expected (gc_pack_rows_f16)")
    ldh = hr.xh.shape[1]
    w = ldh + 8  # row pitch stays a multiple of 16 bytes
    send, full = part.gather_buffers(w, torch.float16, hr.xh.device, tag="half")
    rows = hr.xh.shape[0]
    send[:rows, :ldh].copy_(hr.xh)
    send[:rows, ldh:ldh + 2].copy_(hr.sigma.view(torch.float16).view(rows, 2))
    work = dist.all_gather_into_tensor(full, send, group=group, async_op=async_op)
    out = HalfRows(full[:, :ldh], torch.empty(0), hr.K)

    def finish():
        out.sigma = full[:, ldh:ldh + 2].contiguous().view(torch.float32).view(-1)
        return out

    return out, work, finish


def all_gather_half_multi(hrs: list, extra: torch.Tensor | None, part: RowPartition, group=None):
    """All-gather several fp16 row operands (e.g. one per GAT head, each with
    its own row scales) plus ``extra`` fp32 columns (the GAT target scores
    t) in ONE collective.  Row layout in halves: each operand's ldh halves,
    then the scales and the extra columns as fp32 bit patterns, padded to a
    multiple of 8 halves (16 bytes).  Returns (list of HalfRows over the
    gather buffer, extra_full [world*max_rows, E] fp32)."""
    dev = hrs[0].xh.device
    if any(hr.chunks != 1 for hr in hrs):
        raise ShapeError("all_gather_half_multi: one scale per row expected (gc_pack_rows_f16)")
    offs, o = [], 0
    for hr in hrs:
        offs.append(o)
        o += hr.xh.shape[1]
    n_sc = len(hrs)
    E = 0 if extra is None else extra.shape[1]
    tail = (2 * (n_sc + E) + 7) // 8 * 8
    w = o + tail
    send, full = part.gather_buffers(w, torch.float16, dev, tag=f"halfm{len(hrs)}")
    rows = hrs[0].xh.shape[0]
    if rows:
        for hr, off in zip(hrs, offs):
            send[:rows, off:off + hr.xh.shape[1]].copy_(hr.xh)
        scal = torch.stack([hr.sigma for hr in hrs], 1)
        if E:
            scal = torch.cat([scal, extra.to(torch.float32)], 1)
        send[:rows, o:o + 2 * (n_sc + E)].copy_(scal.contiguous().view(torch.float16))
    dist.all_gather_into_tensor(full, send, group=group)
    scal_full = full[:, o:o + 2 * (n_sc + E)].contiguous().view(torch.float32)
    outs = [HalfRows(full[:, off:off + hr.xh.shape[1]], scal_full[:, i].contiguous(), hr.K)
            for i, (hr, off) in enumerate(zip(hrs, offs))]
    return outs, (scal_full[:, n_sc:].contiguous() if E else None)


def _empty_half(k: int, dev) -> HalfRows:
    ldh = (k + 7) // 8 * 8
    return HalfRows(torch.zeros(0, ldh, dtype=torch.float16, device=dev),
                    torch.zeros(0, dtype=torch.float32, device=dev), k)


def all_gather_rows(x_local: torch.Tensor, part: RowPartition, group=None) -> torch.Tensor:
    """Assemble the full n x k operand from every rank's row block (padded
    all_gather_into_tensor, then the padding is dropped).  Returns a fresh
    tensor (the gather buffer is reused by the next call)."""
    pad = part.max_rows
    full, _ = all_gather_padded(x_local, part, group, tag="rows")
    pieces = [full[p * pad: p * pad + int(part.bounds[p + 1] - part.bounds[p])]
              for p in range(part.world)]
    return torch.cat(pieces, 0)


class CudaOps:
    """The product ops: sm_100a kernels through the C ABI."""

    @staticmethod
    def gemm(a, w, row_scale=None, relu=False, out=None):
        from .sparse import gemm

        return gemm(a, w, row_scale=row_scale, relu=relu, out=out)

    @staticmethod
    def spmm(a: CsrMatrix, b, d_row=None, d_col=None, relu=False, weighted=True, out=None,
             accumulate=False, hub_d=None):
        """``hub_d = (d_row, d_col)``: ``a`` is a unit Ã block or an Ñ = DÃD
        block of a unit Ã, so the hub split (hub.py) may take the dense hub
        columns to the tensor cores (chosen by measurement, cached)."""
        from . import hub
        from .sparse import spmm, spmm_unweighted

        if hub_d is not None:
            pat = a
            vals = a.values if weighted else None
            # fp16 rows carry the unit tail's column scale in their row
            # scales; Ñ's weighted tail keeps it in its values, so only then
            # does the dense part scale its columns
            dcol = hub_d[1] if (weighted or not isinstance(b, HalfRows)) else None
            if weighted:  # Ñ block: the split runs on the unit pattern twin
                key = ("unit_twin",)
                if key not in a._plans:
                    twin = a.with_values(torch.ones_like(a.values))
                    twin._unit = True
                    a._plans[key] = twin
                pat = a._plans[key]
            spec = hub.choose_split(pat, b, dcol, d_row=hub_d[0], values=vals)
            if spec:
                return hub.hybrid_aggregate(pat, b, dcol, spec, d_row=hub_d[0], values=vals,
                                            relu=relu, out=out, accumulate=accumulate)
        if isinstance(b, HalfRows):
            d_col = None  # carried by the row scales
        f = spmm if weighted else spmm_unweighted
        return f(a, b, d_row=d_row, d_col=d_col, relu=relu, out=out, accumulate=accumulate)

    @staticmethod
    def node_scores(x, a_src, a_dst, heads: int, width: int, head_stride: int):
        """s[h], t[h] = X[:, h-block] · a_src[h], · a_dst[h] ([heads, rows])."""
        from .sparse import _ld, _stream

        n = x.shape[0]
        s = torch.empty(heads, n, dtype=torch.float32, device=x.device)
        t = torch.empty(heads, n, dtype=torch.float32, device=x.device)
        if n:
            nat.check(nat.load().gc_node_proj_f32(x.data_ptr(), _ld(x), n, width, heads, head_stride,
                                                  a_src.data_ptr(), a_dst.data_ptr(), s.data_ptr(),
                                                  t.data_ptr(), _stream(x.device)), "node_proj")
        return s, t

    @staticmethod
    def gat_aggregate(a: CsrMatrix, s, t, slope, b, relu=False, out=None):
        from .sparse import gat_aggregate

        return gat_aggregate(a, s, t, slope, b, relu=relu, out=out)

    @staticmethod
    def gat_sddmm_aggregate(a: CsrMatrix, a_src, a_dst, slope, b, b_self, relu=False, out=None):
        from .sparse import gat_sddmm_aggregate

        res = gat_sddmm_aggregate(a, a_src, a_dst, slope, b, relu=relu, out=out, b_self=b_self)
        if res is not None:
            return res
        # outside the fused kernel's range (K % 4, K > 1024, alignment): α by
        # the SDDMM attention kernel, then the weighted SpMM
        from .sparse import spmm

        alpha = CudaOps.attn_sddmm(a, b, b_self, a_src, a_dst, slope, 1, b.shape[1])
        return spmm(a.with_values(alpha[0]), b, relu=relu, out=out)

    @staticmethod
    def attn_sddmm(a: CsrMatrix, hw, hw_self, a_src, a_dst, slope, heads: int, k2: int):
        """α [heads, nnz] of the SDDMM attention (gc_attn_sddmm_f32) on a row
        block: source terms from ``hw_self`` (this rank's rows), target terms
        gathered from ``hw`` (padded layout)."""
        from .sparse import _ld, _stream

        m = a.nnz
        alpha = torch.empty(heads, m, dtype=torch.float32, device=hw.device)
        s_work = torch.empty(heads, max(a.n_rows, 1), dtype=torch.float32, device=hw.device)
        heavy = a.softmax_heavy_rows()
        nat.check(nat.load().gc_attn_sddmm_f32(
            a.row_ptr.data_ptr(), a.col_idx.data_ptr(), hw.data_ptr(), _ld(hw), hw_self.data_ptr(),
            _ld(hw_self), k2, heads, a_src.data_ptr(), a_dst.data_ptr(), float(slope), a.n_rows, m,
            heavy.data_ptr(), heavy.numel(), s_work.data_ptr(), alpha.data_ptr(),
            _stream(hw.device)), "attn_sddmm")
        return alpha


def dist_gcn_layer(part: RowPartition, h_local: torch.Tensor, w: torch.Tensor, *,
                   composition: str, order: str, d: torch.Tensor | None = None,
                   ops=CudaOps, group=None, overlap: bool = False,
                   hub_unit: bool = False) -> torch.Tensor:
    """One GCN layer on this rank's rows (reference gcn.py:125-161 on a row
    block).  ``part.local`` is Ñ's block for precompute or Ã's block for
    dynamic; ``d`` is the FULL D^-1/2 vector (needed for dynamic, and for the
    hub split).  ``hub_unit``: Ã is unit-valued, so the aggregation may use
    the hub split (hub.py) on this rank's block.  Returns this rank's output
    rows.  A rank with no rows still joins the collective and returns a
    0-row output."""
    dyn = composition == "dynamic"
    if dyn and d is None:
        raise ValueError("dynamic composition needs the degree vector")
    hub_unit = hub_unit and d is not None
    d_loc = d[part.lo:part.hi] if (dyn or hub_unit) else None
    weighted = not (dyn and part.local.has_unit_values)
    if ops is CudaOps and _half_gathered(part, w.shape[1] if order == "update_first"
                                         else h_local.shape[1], h_local):
        return _dist_gcn_half(part, h_local, w, dyn, order, d, d_loc, weighted, group,
                              overlap, hub_unit)
    if part.rows == 0:
        src = ops.gemm(h_local, w) if order == "update_first" else h_local
        all_gather_padded(src, part, group)
        return torch.zeros(0, w.shape[1], dtype=torch.float32, device=h_local.device)
    if overlap:
        loc, rem = part.split_local_remote()
        d_pad = part.pad_vector(d) if (dyn or hub_unit) else None
        src = ops.gemm(h_local, w) if order == "update_first" else h_local
        full, work = all_gather_padded(src, part, group, async_op=True)
        # owned-column edges while the gather is in flight
        dl = d_loc if dyn else None
        # (on power-law graphs the owned columns of the first ranks are the
        # hubs: the owned pass may take the dense split as well)
        loc_kw = {"hub_d": (d_loc, d_loc)} if hub_unit else {}
        y = ops.spmm(loc, src, d_row=dl, d_col=dl, relu=False, weighted=weighted, **loc_kw)
        work.wait()
        last = order == "update_first"
        hub_kw = {"hub_d": (d_loc, d_pad)} if hub_unit else {}
        y = ops.spmm(rem, full, d_row=dl, d_col=d_pad if dyn else None, relu=last,
                     weighted=weighted, out=y, accumulate=True, **hub_kw)
        return y if last else ops.gemm(y, w, relu=True)
    pat = part.padded()
    d_pad = part.pad_vector(d) if (dyn or hub_unit) else None
    hub_kw = {"hub_d": (d_loc, d_pad)} if hub_unit else {}
    dl = d_loc if dyn else None
    if order == "update_first":
        full, _ = all_gather_padded(ops.gemm(h_local, w), part, group)
        return ops.spmm(pat, full, d_row=dl, d_col=d_pad if dyn else None, relu=True,
                        weighted=weighted, **hub_kw)
    full, _ = all_gather_padded(h_local, part, group)
    x = ops.spmm(pat, full, d_row=dl, d_col=d_pad if dyn else None, relu=False, weighted=weighted,
                 **hub_kw)
    return ops.gemm(x, w, relu=True)


def _half_gathered(part: RowPartition, k: int, like: torch.Tensor) -> bool:
    """The TF32 class's fp16 gather rows (gcn.half_gather), decided on the
    gathered operand's size so every rank takes the same branch."""
    from . import gcn
    from .sparse import get_gemm_precision

    return (gcn.HALF_GATHER and get_gemm_precision() == "tf32" and like.is_cuda and k % 8 == 0
            and part.world * part.max_rows * k * 4 > gcn.HALF_MIN_BYTES)


def _dist_gcn_half(part, h_local, w, dyn, order, d, d_loc, weighted, group, overlap, hub_unit):
    """dist_gcn_layer in the TF32 class with fp16 gather rows: the local
    operand is packed once (d folded for the dynamic composition), the
    all-gather moves fp16 rows + scales (half the bytes), and every pass
    reads HalfRows."""
    ops = CudaOps
    src = ops.gemm(h_local, w) if order == "update_first" else h_local
    if part.rows == 0:  # still joins the collective
        k = src.shape[1]
        ldh = (k + 7) // 8 * 8
        empty = HalfRows(torch.zeros(0, ldh, dtype=torch.float16, device=src.device),
                         torch.zeros(0, dtype=torch.float32, device=src.device), k)
        _, work, _ = all_gather_half(empty, part, group)
        return torch.zeros(0, w.shape[1], dtype=torch.float32, device=h_local.device)
    hr = pack_rows_f16(src, d_loc if dyn else None)
    dl = d_loc if dyn else None
    last = order == "update_first"
    if overlap:
        loc, rem = part.split_local_remote()
        full, work, finish = all_gather_half(hr, part, group, async_op=True)
        loc_kw = {"hub_d": (d_loc, d_loc)} if hub_unit else {}
        y = ops.spmm(loc, hr, d_row=dl, relu=False, weighted=weighted, **loc_kw)
        work.wait()
        full = finish()
        hub_kw = {"hub_d": (d_loc, part.pad_vector(d))} if hub_unit else {}
        y = ops.spmm(rem, full, d_row=dl, relu=last, weighted=weighted, out=y, accumulate=True,
                     **hub_kw)
        return y if last else ops.gemm(y, w, relu=True)
    full, work, finish = all_gather_half(hr, part, group)
    full = finish()
    hub_kw = {"hub_d": (d_loc, part.pad_vector(d))} if hub_unit else {}
    y = ops.spmm(part.padded(), full, d_row=dl, relu=last, weighted=weighted, **hub_kw)
    return y if last else ops.gemm(y, w, relu=True)


def _pad4(n: int) -> int:
    return (n + 3) // 4 * 4


def dist_gat_layer(part: RowPartition, h_local: torch.Tensor, spec, *, ops=CudaOps,
                   group=None) -> torch.Tensor:
    """One GAT layer (``spec``: a :class:`~.gat.GatLayerSpec`, any heads,
    composition and attention form) on this rank's rows of the unit Ã —
    reference gat.py:121-153 on a row block.  One all-gather per layer of the
    operand in the module table; the aggregation reads the padded gather
    buffer through the remapped pattern.  Returns this rank's output rows
    (rows x heads*k2)."""
    from .gat import AttentionForm, GatComposition, _folded_attention_vectors

    H, k1, k2 = spec.heads, spec.k1, spec.k2
    dev = h_local.device
    if tuple(h_local.shape) != (part.rows, k1):
        raise ShapeError(f"embeddings shape {tuple(h_local.shape)} != ({part.rows}, {k1})")
    relu = spec.activation == "relu"
    slope = spec.leaky_slope
    a_src, a_dst = spec.attn_src.to(dev), spec.attn_dst.to(dev)
    pat = part.padded()
    out = torch.empty(part.rows, k2 * H, dtype=torch.float32, device=dev)
    recompute = spec.composition is GatComposition.RECOMPUTE
    sddmm = spec.attention is AttentionForm.SDDMM
    w = spec.weights
    if not recompute:
        hw = ops.gemm(h_local, w)  # rows x H*k2
        if sddmm:
            full, _ = all_gather_padded(hw, part, group, tag="gat")
            if part.rows == 0:
                return out
            for i in range(H):
                cs = slice(i * k2, (i + 1) * k2)
                ops.gat_sddmm_aggregate(pat, a_src[cs], a_dst[cs], slope, full[:, cs], hw[:, cs],
                                        relu=relu, out=out[:, cs])
            return out
        s, t = ops.node_scores(hw, a_src, a_dst, H, k2, k2)
        if ops is CudaOps and k2 % 8 == 0 and _half_gathered(part, H * k2, hw):
            # TF32 class: per-head fp16 rows + scales and t in one collective
            hrs = [pack_rows_f16(hw[:, i * k2:(i + 1) * k2]) if part.rows else
                   _empty_half(k2, dev) for i in range(H)]
            full_h, t_full = all_gather_half_multi(hrs, t.t() if part.rows else
                                                   torch.zeros(0, H, device=dev), part, group)
            if part.rows == 0:
                return out
            t_full = t_full.t().contiguous()
            for i in range(H):
                cs = slice(i * k2, (i + 1) * k2)
                ops.gat_aggregate(pat, s[i], t_full[i], slope, full_h[i], relu=relu,
                                  out=out[:, cs])
            return out
        wid = H * k2
        full, _ = all_gather_padded(torch.cat([hw, t.t(), hw.new_zeros(hw.shape[0], _pad4(H) - H)],
                                              1), part, group, tag="gat")
        if part.rows == 0:
            return out
        t_full = full[:, wid:wid + H].t().contiguous()
        for i in range(H):
            cs = slice(i * k2, (i + 1) * k2)
            ops.gat_aggregate(pat, s[i], t_full[i], slope, full[:, cs], relu=relu, out=out[:, cs])
        return out
    if sddmm:
        # α from the SDDMM over HW rows, then (α H) W: gather [H_p | H_p W]
        hw = ops.gemm(h_local, w)
        k1p = _pad4(k1)
        parts_ = [h_local] + ([h_local.new_zeros(h_local.shape[0], k1p - k1)] if k1p > k1 else [])             + [hw]
        full, _ = all_gather_padded(torch.cat(parts_, 1), part, group, tag="gat")
        if part.rows == 0:
            return out
        h_full, hw_full = full[:, :k1], full[:, k1p:]
        alpha = ops.attn_sddmm(pat, hw_full, hw, a_src, a_dst, slope, H, k2)
        for i in range(H):
            ah = ops.spmm(pat.with_values(alpha[i]), h_full, relu=False, weighted=True)
            ops.gemm(ah, w[:, i * k2:(i + 1) * k2], relu=relu, out=out[:, i * k2:(i + 1) * k2])
        return out
    # recompute, reassociated scores: s = H (W a_src), t = H (W a_dst) —
    # no HW GEMM; gather [H_p | t_p]
    if ops is CudaOps:
        u, v = _folded_attention_vectors(spec)  # exact-fp32 GEMVs, cached on the spec
    else:
        uv = [ops.gemm(w[:, i * k2:(i + 1) * k2], torch.stack([a_src[i * k2:(i + 1) * k2],
                                                               a_dst[i * k2:(i + 1) * k2]], 1))
              for i in range(H)]
        u = torch.cat([x[:, 0] for x in uv]).contiguous()
        v = torch.cat([x[:, 1] for x in uv]).contiguous()
    s, t = ops.node_scores(h_local, u, v, H, k1, 0)
    if ops is CudaOps and _half_gathered(part, k1, h_local):
        # TF32 class: fp16 rows of H + scales and t in one collective
        hr = pack_rows_f16(h_local) if part.rows else _empty_half(k1, dev)
        full_h, t_full = all_gather_half_multi([hr], t.t() if part.rows else
                                               torch.zeros(0, H, device=dev), part, group)
        if part.rows == 0:
            return out
        t_full = t_full.t().contiguous()
        for i in range(H):
            ah = ops.gat_aggregate(pat, s[i], t_full[i], slope, full_h[0], relu=False)
            ops.gemm(ah, w[:, i * k2:(i + 1) * k2], relu=relu, out=out[:, i * k2:(i + 1) * k2])
        return out
    full, _ = all_gather_padded(torch.cat([h_local, t.t(), h_local.new_zeros(h_local.shape[0],
                                                                             _pad4(k1 + H) - k1 - H)],
                                          1), part, group, tag="gat")
    if part.rows == 0:
        return out
    h_full = full[:, :k1]
    t_full = full[:, k1:k1 + H].t().contiguous()
    for i in range(H):
        ah = ops.gat_aggregate(pat, s[i], t_full[i], slope, h_full, relu=False)
        ops.gemm(ah, w[:, i * k2:(i + 1) * k2], relu=relu, out=out[:, i * k2:(i + 1) * k2])
    return out
