"""Row-partitioned layers across GPUs.

One process per GPU (``torch.distributed``, NCCL over NVLink on the box,
gloo in the CPU tests).  Ã is cut into contiguous, nnz-balanced row blocks
(``partition_rows`` — the C-ABI host function, bit-exact with the oracle);
rank p owns rows [b_p, b_{p+1}) with global column ids.  Per layer exactly one
all-gather assembles the operand the local SpMM gathers:

    composition              all-gathered operand
    GCN A(HW)                (H_p W)          (d ⊙ folded into the SpMM gather)
    GCN (AH)W                H_p
    GAT reuse                H_p W and t_p
    GAT recompute            H_p and t_p (+ H_p W for the local attention)

Output rows stay partitioned and feed the next layer.  Blocks are padded to
the largest block for ``all_gather_into_tensor``.

Overlap (``overlap=True``): the local block of the
pattern is split by column into the edges whose source row this rank owns
(aggregated straight from its own operand block, while the all-gather is in
flight) and the remote edges (column ids remapped into the padded gather
buffer, so no unpad copy).  The remote pass accumulates into the local one
(``out += d_i * acc``; ReLU on the total).

The compute ops are injectable (``ops``) so the host logic — partition,
padding, gather, unpad, assembly — is testable on CPU with gloo and the
oracle standing in for the CUDA kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat
from .sparse import CsrMatrix


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
        return int(np.diff(self.bounds).max())

    @classmethod
    def of(cls, a: CsrMatrix, rank: int, world: int) -> "RowPartition":
        b = partition_rows(a.row_ptr, world)
        return cls(rank, world, b, a.take_rows(int(b[rank]), int(b[rank + 1])))

    def split_local_remote(self) -> tuple[CsrMatrix, CsrMatrix]:
        """(edges from owned rows, columns rebased to the local block;
        remaining edges, columns remapped into the padded gather buffer)."""
        if getattr(self, "_lr", None) is None:
            a = self.local
            col = a.col_idx.long()
            rows = a.row_of_nnz()
            own = (col >= self.lo) & (col < self.hi)
            bounds = torch.as_tensor(self.bounds, device=col.device)
            owner = torch.searchsorted(bounds[1:], col, right=True)
            padded = owner * self.max_rows + (col - bounds[owner])

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


def all_gather_padded(x_local: torch.Tensor, part: RowPartition, group=None, async_op=False):
    """Padded all-gather: returns (buffer of world*max_rows rows, work handle)."""
    k = x_local.shape[1]
    pad = part.max_rows
    if x_local.shape[0] == pad:
        buf = x_local.contiguous()
    else:
        buf = torch.zeros(pad, k, dtype=x_local.dtype, device=x_local.device)
        buf[: x_local.shape[0]] = x_local
    full = torch.empty(part.world * pad, k, dtype=x_local.dtype, device=x_local.device)
    work = dist.all_gather_into_tensor(full, buf, group=group, async_op=async_op)
    return full, work


def all_gather_rows(x_local: torch.Tensor, part: RowPartition, group=None) -> torch.Tensor:
    """Assemble the full n x k operand from every rank's row block (padded
    all_gather_into_tensor, then the padding is dropped)."""
    pad = part.max_rows
    full, _ = all_gather_padded(x_local, part, group)
    if all(int(part.bounds[p + 1] - part.bounds[p]) == pad for p in range(part.world)):
        return full
    pieces = [full[p * pad: p * pad + int(part.bounds[p + 1] - part.bounds[p])]
              for p in range(part.world)]
    return torch.cat(pieces, 0)


class CudaOps:
    """The product ops: sm_100a kernels through the C ABI."""

    @staticmethod
    def gemm(a, w, row_scale=None, relu=False):
        from .sparse import gemm

        return gemm(a, w, row_scale=row_scale, relu=relu)

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
            if weighted:  # Ñ block: the split runs on the unit pattern twin
                key = ("unit_twin",)
                if key not in a._plans:
                    twin = a.with_values(torch.ones_like(a.values))
                    twin._unit = True
                    a._plans[key] = twin
                pat = a._plans[key]
            spec = hub.choose_split(pat, b, hub_d[1], d_row=hub_d[0], values=vals)
            if spec:
                return hub.hybrid_aggregate(pat, b, hub_d[1], spec, d_row=hub_d[0], values=vals,
                                            relu=relu, out=out, accumulate=accumulate)
        f = spmm if weighted else spmm_unweighted
        return f(a, b, d_row=d_row, d_col=d_col, relu=relu, out=out, accumulate=accumulate)


def dist_gcn_layer(part: RowPartition, h_local: torch.Tensor, w: torch.Tensor, *,
                   composition: str, order: str, d: torch.Tensor | None = None,
                   ops=CudaOps, group=None, overlap: bool = False,
                   hub_unit: bool = False) -> torch.Tensor:
    """One GCN layer on this rank's rows.  ``part.local`` is Ñ's block for
    precompute or Ã's block for dynamic; ``d`` is the FULL D^-1/2 vector
    (needed for dynamic, and for the hub split).  ``hub_unit``: Ã is
    unit-valued, so the aggregation may use the hub split (hub.py) on this
    rank's block.  Returns this rank's output rows."""
    dyn = composition == "dynamic"
    if dyn and d is None:
        raise ValueError("dynamic composition needs the degree vector")
    hub_unit = hub_unit and d is not None
    d_loc = d[part.lo:part.hi] if (dyn or hub_unit) else None
    weighted = not (dyn and part.local.has_unit_values)
    if overlap:
        loc, rem = part.split_local_remote()
        d_pad = None
        if dyn or hub_unit:
            d_pad = torch.zeros(part.world * part.max_rows, dtype=d.dtype, device=d.device)
            for p in range(part.world):
                lo, hi = int(part.bounds[p]), int(part.bounds[p + 1])
                d_pad[p * part.max_rows: p * part.max_rows + hi - lo] = d[lo:hi]
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
    hub_kw = {"hub_d": (d_loc, d)} if hub_unit else {}
    dl = d_loc if dyn else None
    if order == "update_first":
        hw_loc = ops.gemm(h_local, w)
        hw = all_gather_rows(hw_loc, part, group)
        return ops.spmm(part.local, hw, d_row=dl, d_col=d if dyn else None, relu=True,
                        weighted=weighted, **hub_kw)
    h = all_gather_rows(h_local, part, group)
    x = ops.spmm(part.local, h, d_row=dl, d_col=d if dyn else None, relu=False, weighted=weighted,
                 **hub_kw)
    return ops.gemm(x, w, relu=True)
