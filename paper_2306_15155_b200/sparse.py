"""CSR / dense types and the primitive kernels every layer composition uses.

Drop-in mirror of ``gnncompose/sparse.py`` (reference 0.1.0): same names,
argument meaning and exception types.  Differences, all B200-driven:

* storage is on the GPU (torch tensors): indices int32, values float32;
* every compute primitive calls a hand-written sm_100a kernel through the C
  ABI (``include/gnnc.h``); there is no CPU fallback — calling one with CPU
  tensors raises;
* numpy inputs are accepted (uploaded) and numpy outputs returned, so code
  written against the reference keeps working; torch CUDA tensors in give
  torch CUDA tensors out with no host round trip;
* extensions the layer code uses: fused ``d_row``/``d_col`` degree scaling and
  ``relu`` epilogues, an nnz-split plan for power-law rows.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat


class ShapeError(ValueError):
    """Operand dimensions do not conform (reference sparse.py:17)."""


class DegenerateNodeError(ValueError):
    """A node violates a degree precondition, e.g. a zero-degree row (sparse.py:21)."""


# ---------------------------------------------------------------------------
# device / operand plumbing
# ---------------------------------------------------------------------------


def default_device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
        else torch.device("cpu")


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _require_cuda(*ts: torch.Tensor | None) -> torch.device:
    dev = None
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise RuntimeError(
                "gnnc kernels run on the GPU only (no CPU fallback); got a CPU tensor")
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise ValueError(f"operands on different devices: {dev} vs {t.device}")
    if dev is None:
        raise RuntimeError("no CUDA operand")
    return dev


def dense_matrix(data) -> torch.Tensor:
    """Coerce to a row-major float32 2-D tensor and check all entries are finite
    (reference sparse.py:25-32)."""
    t = torch.as_tensor(np.asarray(data) if not isinstance(data, torch.Tensor) else data)
    t = t.to(torch.float32).contiguous()
    if t.dim() != 2:
        raise ShapeError(f"dense matrix must be 2-D, got ndim={t.dim()}")
    if not bool(torch.isfinite(t).all()):
        raise ValueError("dense matrix contains non-finite entries")
    return t


class _Operand:
    """A dense 2-D float32 CUDA operand plus where it came from.

    numpy in -> numpy out (the reference's ndarray return type); a CPU torch
    tensor in (ideally pinned) -> a pinned CPU tensor out; a CUDA tensor in ->
    CUDA tensor out with no host traffic."""

    __slots__ = ("t", "host", "kind")

    def __init__(self, b, device: torch.device, what: str = "dense operand"):
        if isinstance(b, torch.Tensor) and (b.is_cuda or device.type != "cuda"):
            self.host, self.kind = False, "device"
            t = b if b.dtype == torch.float32 else b.float()
            if t.device != device:
                t = t.to(device)
        else:
            self.host = True
            if isinstance(b, torch.Tensor):
                self.kind = "torch"
                t = b if b.dtype == torch.float32 else b.float()
            else:
                self.kind = "numpy"
                t = torch.from_numpy(np.ascontiguousarray(np.asarray(b), dtype=np.float32))
            if t.dim() == 2 and t.stride(1) != 1:
                t = t.contiguous()
            t = t.to(device, non_blocking=t.is_pinned())
        if t.dim() != 2:
            raise ShapeError(f"{what} must be 2-D, got ndim={t.dim()}")
        if t.stride(1) != 1 or (t.size(0) > 1 and t.stride(0) < t.size(1)):
            t = t.contiguous()
        self.t = t

    def wrap(self, out: torch.Tensor):
        if not self.host:
            return out
        if self.kind == "numpy":
            return out.cpu().numpy()
        dst = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        dst.copy_(out, non_blocking=True)
        torch.cuda.current_stream(out.device).synchronize()
        return dst


# ---- optional CUDA-event timing of individual kernel calls (bench.py) -------
_TIMERS: dict[str, list] | None = None


class kernel_timing:
    """Context manager: record a CUDA event pair around every call of the named
    primitives ("spmm", "gemm", "sddmm_norm", "attention") on the stream the
    kernel is launched on.  ``durations_ms(name)`` after a synchronize."""

    def __init__(self, *names: str):
        self.names = names
        self.events: dict[str, list] = {n: [] for n in names}

    def __enter__(self):
        global _TIMERS
        _TIMERS = self.events
        return self

    def __exit__(self, *exc):
        global _TIMERS
        _TIMERS = None

    def durations_ms(self, name: str) -> list[float]:
        return [a.elapsed_time(b) for a, b in self.events[name]]


def _timed_call(name: str, dev: torch.device, fn):
    ev = _TIMERS.get(name) if _TIMERS is not None else None
    if ev is None:
        return fn()
    st = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    rc = fn()
    b.record(st)
    ev.append((a, b))
    return rc


def _ld(t: torch.Tensor) -> int:
    return t.stride(0) if t.size(0) > 1 else max(t.size(1), 1)


# ---------------------------------------------------------------------------
# CsrMatrix — reference sparse.py:43-188
# ---------------------------------------------------------------------------


class CsrMatrix:
    """Sparse matrix in compressed-row form, resident on one device.

    Invariants (checked at construction unless ``validate=False``), as in the
    reference: ``row_ptr[0] == 0``, ``row_ptr[n_rows] == nnz``, non-decreasing;
    column indices strictly increasing within each row and ``< n_cols``;
    ``len(values) == len(col_idx)``.  Instances are immutable after
    construction.
    """

    def __init__(self, n_rows: int, n_cols: int, row_ptr, col_idx, values, validate: bool = True,
                 device: torch.device | str | None = None):
        dev = torch.device(device) if device is not None else None
        if dev is None:
            dev = next((x.device for x in (row_ptr, col_idx, values) if isinstance(x, torch.Tensor)),
                       default_device())
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_ptr = _as_index(row_ptr, dev)
        self.col_idx = _as_index(col_idx, dev)
        self.values = _as_values(values, dev)
        self._unit: bool | None = None
        self._plans: dict = {}
        self._dmax: int | None = None
        if validate:
            self._check()

    # -- validation (sparse.py:74-98) ---------------------------------------
    def _check(self):
        if self.n_rows < 0 or self.n_cols < 0:
            raise ShapeError("matrix dimensions must be non-negative")
        if self.n_rows >= 2**31 - 1 or self.n_cols >= 2**31 - 1 or self.col_idx.numel() >= 2**31 - 1:
            raise ShapeError("int32 index range exceeded")
        if tuple(self.row_ptr.shape) != (self.n_rows + 1,):
            raise ShapeError(f"row_ptr length {self.row_ptr.numel()} != n_rows+1 = {self.n_rows + 1}")
        rp = self.row_ptr
        if int(rp[0]) != 0 or int(rp[-1]) != self.col_idx.numel():
            raise ShapeError("row_ptr must start at 0 and end at nnz")
        if self.n_rows and bool((rp[1:] < rp[:-1]).any()):
            raise ShapeError("row_ptr must be non-decreasing")
        if self.values.shape != self.col_idx.shape:
            raise ShapeError("values and col_idx must have equal length")
        ci = self.col_idx
        if ci.numel():
            if int(ci.min()) < 0 or int(ci.max()) >= self.n_cols:
                raise ShapeError("column index out of range")
            d = ci[1:] - ci[:-1]
            boundary = torch.zeros(d.numel(), dtype=torch.bool, device=ci.device)
            starts = rp[1:-1].long()
            starts = starts[(starts > 0) & (starts <= d.numel())]
            boundary[starts - 1] = True
            if not bool(((d > 0) | boundary).all()):
                raise ShapeError("column indices must be strictly increasing per row")

    # -- construction helpers ----------------------------------------------------
    @classmethod
    def from_dense(cls, arr, device=None) -> "CsrMatrix":
        a = torch.as_tensor(np.asarray(arr, dtype=np.float64) if not isinstance(arr, torch.Tensor)
                            else arr)
        if a.dim() != 2:
            raise ShapeError("from_dense expects a 2-D array")
        dev = torch.device(device) if device is not None else default_device()
        a = a.to(dev)
        nz = torch.nonzero(a, as_tuple=True)
        counts = torch.bincount(nz[0], minlength=a.shape[0])
        row_ptr = torch.cat([counts.new_zeros(1), torch.cumsum(counts, 0)])
        return cls(a.shape[0], a.shape[1], row_ptr, nz[1], a[nz], device=dev)

    @classmethod
    def from_coo(cls, n_rows: int, n_cols: int, rows, cols, values, sum_duplicates: bool = True,
                 device=None) -> "CsrMatrix":
        """Build from unordered coordinate triplets; duplicate entries are summed
        (reference sparse.py:120-146: lexsort by (row, col) then reduceat).

        The index arrays come out bit-identical to the reference (the CSR of a
        set of distinct coordinates is unique).  Duplicate values are summed in
        float64 before rounding to float32."""
        dev = torch.device(device) if device is not None else default_device()
        r = torch.as_tensor(rows).to(dev, torch.int64).reshape(-1)
        c = torch.as_tensor(cols).to(dev, torch.int64).reshape(-1)
        v = torch.as_tensor(np.asarray(values, dtype=np.float64) if not isinstance(values, torch.Tensor)
                            else values).to(dev, torch.float64).reshape(-1)
        if not (r.shape == c.shape == v.shape):
            raise ShapeError("rows/cols/values must have equal length")
        # range checks before the (row, col) key is formed: an out-of-range
        # column would otherwise alias a valid entry of the next row and be
        # summed into it (the reference lexsorts and raises in _check)
        # (rows first: the reference's row_ptr-length check precedes the
        # column check)
        if r.numel():
            if int(r.min()) < 0 or int(r.max()) >= int(n_rows):
                raise ShapeError("row index out of range")
            if int(c.min()) < 0 or int(c.max()) >= int(n_cols):
                raise ShapeError("column index out of range")
        key = r * max(int(n_cols), 1) + c
        key, order = torch.sort(key, stable=True)
        r, c, v = r[order], c[order], v[order]
        if sum_duplicates and r.numel():
            first = torch.ones(r.numel(), dtype=torch.bool, device=dev)
            first[1:] = key[1:] != key[:-1]
            if not bool(first.all()):
                seg = torch.cumsum(first.long(), 0) - 1
                starts = torch.nonzero(first).reshape(-1)
                if dev.type == "cpu":  # sequential sums, exactly np.add.reduceat
                    vs = torch.from_numpy(np.add.reduceat(v.numpy(), starts.numpy()))
                else:
                    vs = torch.zeros(starts.numel(), dtype=torch.float64, device=dev)
                    vs.index_add_(0, seg, v)
                r, c, v = r[starts], c[starts], vs
        counts = torch.bincount(r, minlength=int(n_rows))
        row_ptr = torch.cat([counts.new_zeros(1), torch.cumsum(counts, 0)])
        return cls(n_rows, n_cols, row_ptr, c, v, device=dev)

    def with_values(self, values, validate: bool = False) -> "CsrMatrix":
        """Same sparsity pattern (shared row_ptr/col_idx), new values."""
        v = _as_values(values, self.device)
        if v.shape != self.col_idx.shape:
            raise ShapeError("replacement values must match nnz")
        out = CsrMatrix.__new__(CsrMatrix)
        out.n_rows, out.n_cols = self.n_rows, self.n_cols
        out.row_ptr, out.col_idx, out.values = self.row_ptr, self.col_idx, v
        out._unit, out._plans, out._dmax = None, self._plans, self._dmax  # plans depend on pattern only
        if validate:
            out._check()
        return out

    # -- binary CSR file ----------------------------------
    # The reference ingests graphs only through MatrixMarket text
    # (mtxio.py), which parses at a few M entries/s; a graph the size of
    # Reddit takes minutes.  ``.gcsr`` stores the device layout verbatim so a
    # load is a memory map + one host->device copy per array:
    #   bytes 0..63   header: b"GCSR" + u32 version, i64 n_rows, i64 n_cols,
    #                 i64 nnz, u32 flags (bit 0: unit values, not stored),
    #                 zero padding
    #   then          row_ptr int32[n_rows+1], col_idx int32[nnz],
    #                 values float32[nnz] (absent if unit), each section
    #                 starting on a 64-byte boundary, little-endian.
    GCSR_MAGIC = b"GCSR"
    GCSR_VERSION = 1

    def save(self, path) -> None:
        """Write the matrix as a ``.gcsr`` file (layout above)."""
        unit = self.has_unit_values
        head = np.zeros(64, dtype=np.uint8)
        hdr = (self.GCSR_MAGIC + np.array([self.GCSR_VERSION], "<u4").tobytes()
               + np.array([self.n_rows, self.n_cols, self.nnz], "<i8").tobytes()
               + np.array([1 if unit else 0], "<u4").tobytes())
        head[:len(hdr)] = np.frombuffer(hdr, np.uint8)
        sections = [self.row_ptr.cpu().numpy().astype("<i4", copy=False),
                    self.col_idx.cpu().numpy().astype("<i4", copy=False)]
        if not unit:
            sections.append(self.values.cpu().numpy().astype("<f4", copy=False))
        with open(path, "wb") as f:
            f.write(head.tobytes())
            for arr in sections:
                f.write(arr.tobytes())
                pad = (-arr.nbytes) % 64
                if pad:
                    f.write(b"\0" * pad)

    @classmethod
    def _gcsr_header(cls, path):
        if os.path.getsize(path) < 64:
            raise ShapeError(f"{path}: not a .gcsr file (shorter than its header)")
        raw = np.memmap(path, dtype=np.uint8, mode="r")
        if bytes(raw[:4]) != cls.GCSR_MAGIC:
            raise ShapeError(f"{path}: not a .gcsr file")
        version = int(raw[4:8].view("<u4")[0])
        if version != cls.GCSR_VERSION:
            raise ShapeError(f"{path}: unsupported .gcsr version {version}")
        n_rows, n_cols, nnz = (int(x) for x in raw[8:32].view("<i8"))
        flags = int(raw[32:36].view("<u4")[0])
        if min(n_rows, n_cols, nnz) < 0:
            raise ShapeError(f"{path}: negative dimension in header")
        rp_bytes = 4 * (n_rows + 1)
        ci_off = 64 + rp_bytes + (-rp_bytes) % 64
        va_off = ci_off + 4 * nnz + (-4 * nnz) % 64
        unit = bool(flags & 1)
        need = (ci_off + 4 * nnz) if unit else (va_off + 4 * nnz)
        if raw.size < need:
            raise ShapeError(f"{path}: truncated .gcsr file")
        return raw, n_rows, n_cols, nnz, unit, ci_off, va_off

    @classmethod
    def read_row_ptr(cls, path) -> np.ndarray:
        """The row_ptr of a ``.gcsr`` file as a host int64 array (O(n) bytes
        read; col_idx / values are not touched)."""
        raw, n_rows, *_ = cls._gcsr_header(path)
        return raw[64:64 + 4 * (n_rows + 1)].view("<i4").astype(np.int64)

    @classmethod
    def load(cls, path, device=None, validate: bool = True,
             rows: tuple[int, int] | None = None) -> "CsrMatrix":
        """Read a ``.gcsr`` file written by :meth:`save` onto ``device``.
        ``rows=(lo, hi)`` reads only that row block (rebased row_ptr, global
        column ids — a partition's local adjacency): only those rows' bytes of
        col_idx / values are read.  Truncated or foreign files raise
        ``ShapeError``; the CSR invariants are checked on the device unless
        ``validate=False``."""
        dev = torch.device(device) if device is not None else default_device()
        raw, n_rows, n_cols, nnz, unit, ci_off, va_off = cls._gcsr_header(path)
        lo, hi = (0, n_rows) if rows is None else (int(rows[0]), int(rows[1]))
        if not 0 <= lo <= hi <= n_rows:
            raise ShapeError(f"{path}: row range [{lo}, {hi}) outside [0, {n_rows})")
        rp_host = np.array(raw[64 + 4 * lo:64 + 4 * (hi + 1)].view("<i4"), copy=True)
        b, e = int(rp_host[0]), int(rp_host[-1])
        if not 0 <= b <= e <= nnz:
            raise ShapeError(f"{path}: corrupt row_ptr")

        def section(off: int, dt: str) -> torch.Tensor:
            host = torch.from_numpy(np.array(raw[off + 4 * b:off + 4 * e].view(dt), copy=True))
            return host.to(dev, non_blocking=False)

        rp = torch.from_numpy(rp_host - b).to(dev)
        ci = section(ci_off, "<i4")
        va = torch.ones(e - b, dtype=torch.float32, device=dev) if unit else section(va_off, "<f4")
        out = cls(hi - lo, n_cols, rp, ci, va, validate=validate, device=dev)
        if unit:
            out._unit = True
        return out

    def to(self, device) -> "CsrMatrix":
        dev = torch.device(device)
        out = CsrMatrix(self.n_rows, self.n_cols, self.row_ptr.to(dev), self.col_idx.to(dev),
                        self.values.to(dev), validate=False, device=dev)
        out._unit, out._dmax = self._unit, self._dmax
        return out

    # -- queries -----------------------------------------------------------------
    @property
    def device(self) -> torch.device:
        return self.col_idx.device

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @property
    def has_unit_values(self) -> bool:
        """True iff every stored value is 1 (sparse.py:70-72).  Computed once,
        lazily, to keep the O(nnz) scan off the per-layer hot path."""
        if self._unit is None:
            self._unit = bool(self.values.numel() == 0 or bool((self.values == 1.0).all()))
        return self._unit

    def degrees(self) -> torch.Tensor:
        """Structural per-row non-zero counts (int64)."""
        return (self.row_ptr[1:] - self.row_ptr[:-1]).long()

    def max_degree(self) -> int:
        if self._dmax is None:
            self._dmax = int(self.degrees().max()) if self.n_rows else 0
        return self._dmax

    def row_of_nnz(self) -> torch.Tensor:
        return torch.repeat_interleave(torch.arange(self.n_rows, device=self.device),
                                       self.degrees())

    def to_dense(self) -> torch.Tensor:
        out = torch.zeros(self.n_rows, self.n_cols, dtype=torch.float32, device=self.device)
        out[self.row_of_nnz(), self.col_idx.long()] = self.values
        return out

    def same_pattern(self, other: "CsrMatrix") -> bool:
        return (self.n_rows == other.n_rows and self.n_cols == other.n_cols
                and torch.equal(self.row_ptr, other.row_ptr.to(self.device))
                and torch.equal(self.col_idx, other.col_idx.to(self.device)))

    def numpy(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Host copies (int64 indices, float64 values) — the reference's dtypes."""
        return (self.row_ptr.cpu().numpy().astype(np.int64), self.col_idx.cpu().numpy().astype(np.int64),
                self.values.cpu().numpy().astype(np.float64))

    def take_rows(self, lo: int, hi: int) -> "CsrMatrix":
        """Contiguous row block [lo, hi) with global column ids (a partition's
        local adjacency); row_ptr is rebased."""
        rp = self.row_ptr[lo:hi + 1]
        b, e = int(rp[0]), int(rp[-1])
        return CsrMatrix(hi - lo, self.n_cols, rp - b, self.col_idx[b:e], self.values[b:e],
                         validate=False, device=self.device)

    # -- nnz-split plan (cached per pattern) ----------------------------------------
    def spmm_plan(self, chunk: int, length_classes: bool = True):
        """Work items for GC_SPMM_NNZ_SPLIT: heavy rows (> chunk edges) are cut
        into chunk-sized pieces whose partial sums are combined in fixed order;
        items are ordered longest-length-class first."""
        key = ("split", int(chunk), bool(length_classes))
        if key not in self._plans:
            lib = nat.load()
            rp = np.ascontiguousarray(self.row_ptr.cpu().numpy(), dtype=np.int32)
            ni, ns, nsr = (np.zeros(1, np.int64) for _ in range(3))
            nat.check(lib.gc_spmm_plan_count(rp.ctypes.data, self.n_rows, int(chunk),
                                             ni.ctypes.data_as(nat._i64p), ns.ctypes.data_as(nat._i64p),
                                             nsr.ctypes.data_as(nat._i64p)), "gc_spmm_plan_count")
            items = np.empty((int(ni[0]), 4), np.int32)
            split = np.empty((max(int(nsr[0]), 1), 4), np.int32)
            nat.check(lib.gc_spmm_plan_fill(rp.ctypes.data, self.n_rows, int(chunk),
                                            nat.GC_PLAN_LENGTH_CLASSES if length_classes else 0,
                                            items.ctypes.data, split.ctypes.data), "gc_spmm_plan_fill")
            self._plans[key] = (torch.from_numpy(items).to(self.device),
                                torch.from_numpy(split[: int(nsr[0])]).to(self.device), int(ns[0]))
        return self._plans[key]

    def softmax_heavy_rows(self) -> torch.Tensor:
        """Rows longer than the edge-softmax lane-group threshold (int32, on the
        device, cached per pattern): each gets a whole CTA in the softmax."""
        key = ("softmax_heavy",)
        if key not in self._plans:
            th = nat.load().gc_edge_softmax_heavy_threshold(self.n_rows, self.nnz)
            deg = self.row_ptr[1:] - self.row_ptr[:-1]
            self._plans[key] = torch.nonzero(deg > th).flatten().to(torch.int32).contiguous()
        return self._plans[key]

    def hub_tagged_cols(self, K: int, budget_bytes: int | None = None) -> torch.Tensor:
        """col_idx with the most-referenced columns tagged in bit 31, sized so
        the tagged rows of a K-wide operand fit one SM's L1 (cached)."""
        budget = budget_bytes or HUB_L1_BUDGET
        n_hot = max(1, min(self.n_cols, budget // (4 * max(K, 1))))
        key = ("hub", n_hot)
        if key not in self._plans:
            counts = torch.bincount(self.col_idx.long(), minlength=self.n_cols)
            hot = torch.zeros(self.n_cols, dtype=torch.uint8, device=self.device)
            hot[torch.topk(counts, n_hot).indices] = 1
            tagged = torch.empty_like(self.col_idx)
            nat.check(nat.load().gc_tag_hub_columns(self.col_idx.data_ptr(), self.nnz, hot.data_ptr(),
                                                    tagged.data_ptr(), _stream(self.device)),
                      "tag_hub_columns")
            self._plans[key] = tagged
        return self._plans[key]

    def __repr__(self):
        return f"CsrMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz}, device={self.device})"


def _as_index(x, dev) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64))
    if t.numel() and (int(t.max()) >= 2**31 or int(t.min()) < -(2**31)):
        raise ShapeError("index exceeds int32 range")
    return t.to(dev, torch.int32).contiguous()


def _as_values(x, dev) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    return t.to(dev, torch.float32).contiguous()


# ---------------------------------------------------------------------------
# SpMM — reference sparse.py:240-264
# ---------------------------------------------------------------------------

SPLIT_CHUNK = int(os.environ.get("GNNC_SPLIT_CHUNK", "0"))  # 0: per-launch default
PLAN_MIN_NNZ = 1 << 16  # below this a row-per-group launch needs no plan
# fused aggregate-then-update (spmm_gemm) for narrow updates on graphs small
# enough that the plain lane-group SpMM needs no nnz-split plan (GNNC_SPMM_GEMM=0
# keeps the two-kernel form)
SPMM_GEMM = os.environ.get("GNNC_SPMM_GEMM", "1") != "0"
# GEMM epilogue emitting fp16 rows with one scale per 256-column chunk for
# N > 256 (GNNC_F16ROWS_CHUNKED=0: fp32 product, then a per-row pack)
F16ROWS_CHUNKED = os.environ.get("GNNC_F16ROWS_CHUNKED", "1") != "0"
SPMM_GEMM_MAX_DEG = 1024  # one lane group per row: no heavy-row splitting
# L1 policy tags on hub columns: "0" off, "1" on, "auto" (default): measured
# once per (pattern, K) on the first large launch and cached — the tags win on
# graphs whose hubs fit L1 (arxiv-like) and lose where L2 reuse already
# dominates (Reddit-like), see profiles/spmm_variants.py.
HUB_HINTS = os.environ.get("GNNC_HUB_HINTS", "auto")
HUB_AUTOTUNE_MIN_NNZ = 1 << 20
HUB_L1_BUDGET = int(os.environ.get("GNNC_HUB_L1_BUDGET", str(160 * 1024)))


def _sm_count(dev: torch.device) -> int:
    return torch.cuda.get_device_properties(dev).multi_processor_count


def _plan_args(a: CsrMatrix, K: int, algo: str, dev, gat: bool = False, heads: int = 1):
    """(code, items, n_items, split, n_split, workspace) for one launch."""
    chunk = SPLIT_CHUNK or int(nat.load().gc_spmm_default_chunk(a.n_rows, a.nnz, K, _sm_count(dev)))
    use_split = algo == "split" or (algo == "auto" and a.nnz and (
        a.nnz >= PLAN_MIN_NNZ or a.max_degree() > chunk))
    if not use_split:
        return nat.GC_SPMM_ROW, None, 0, None, 0, None
    items, split, n_slots = a.spmm_plan(chunk)
    ws = None
    if n_slots:
        per_slot = K + (2 * heads if gat else 0)  # partial row (+ (max, sum) per GAT head)
        ws = torch.empty(n_slots * per_slot + (2 if gat else 0), dtype=torch.float32, device=dev)
    return nat.GC_SPMM_NNZ_SPLIT, items, items.shape[0], split, split.shape[0], ws


SPMM_SHRINK = os.environ.get("GNNC_SPMM_SHRINK", "auto")  # lane-group variant: auto | 0 | 1 | 2


def _shrink_candidates(K: int, mode: str = "spmm") -> list[int]:
    if mode in ("gatsd", "gatsdh") and K > 256:
        return [0]  # one wide lane-group shape only (whole row per pass)
    if mode.endswith("h"):  # fp16 rows: lane groups of 16-byte chunks
        return [0] if K <= 16 else ([0, 1] if K <= 32 else [0, 1, 2])
    return [0] if K <= 8 else ([0, 1] if K <= 16 else [0, 1, 2])


def _variant(a: CsrMatrix, K: int, mode: str, probe) -> tuple[bool, int]:
    """Kernel variant for (pattern, K, mode): hub-column L1 tags on/off and the
    lane-group shape.  ``probe(cols, extra_flags)`` runs the kernel into a
    scratch output.  In "auto" mode every candidate is timed once (CUDA
    events, median of 3 after a warm launch) on the first large launch and the
    fastest is cached — the GPU counterpart of the reference's OPT autotuner
    (tiling.py:311-364), over kernel variants instead of CPU tile sizes."""
    hint_mode = HUB_HINTS if isinstance(HUB_HINTS, str) else ("1" if HUB_HINTS else "0")
    shrink_mode = str(SPMM_SHRINK)
    if a.nnz < PLAN_MIN_NNZ:
        return False, 0
    hints = [False, True] if hint_mode == "auto" else [hint_mode == "1"]
    if mode.endswith("h"):
        hints = [False]  # no L1-tag variant with fp16 operand rows
    shrinks = _shrink_candidates(K, mode) if shrink_mode == "auto" else [int(shrink_mode)]
    if len(hints) * len(shrinks) == 1:
        return hints[0], shrinks[0]
    if a.nnz < HUB_AUTOTUNE_MIN_NNZ:
        return (False if hint_mode == "auto" else hints[0]), (0 if shrink_mode == "auto" else shrinks[0])
    key = ("variant", mode, int(K))
    if key not in a._plans:
        times = {}
        for hv in hints:
            cols = a.hub_tagged_cols(K) if hv else a.col_idx
            for sv in shrinks:
                extra = (nat.GC_HUB_TAGGED if hv else 0) | nat.GC_SPMM_SHRINK(sv)
                probe(cols, extra)  # warm
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(3)]
                for e0, e1 in ev:
                    e0.record()
                    probe(cols, extra)
                    e1.record()
                torch.cuda.synchronize()
                times[(hv, sv)] = sorted(e0.elapsed_time(e1) for e0, e1 in ev)[1]
        base = times.get((False, 0), min(times.values()))
        best = min(times, key=times.get)
        # keep the default unless a variant is clearly (>3%) faster
        a._plans[key] = best if times[best] < 0.97 * base else (False, 0)
        a._plans[key + ("times",)] = {f"hints={h},shrink={v}": round(t, 4) for (h, v), t in times.items()}
    return a._plans[key]


def gat_sddmm_aggregate(a: CsrMatrix, a_src: torch.Tensor, a_dst: torch.Tensor, slope: float, b,
                        *, relu: bool = False, out=None, algo: str = "auto", b_self=None):
    """GAT reuse aggregation with SDDMM attention fused in: per edge the
    gathered row B_j gives both e = LeakyReLU(a_src.B_i + a_dst.B_j) and the
    aggregated term (one gather per edge; α never written).  ``b_self``: the
    rows B_i of the pattern's own rows when ``a`` is a row block (a rank's
    rows of a partitioned graph, B the gathered operand); default ``b`` with a
    square pattern.  Returns None when the operand shape is outside the
    kernel's range (K > 1024, unaligned)."""
    dev = a.device
    half = isinstance(b, HalfRows)
    bt = b.xh if half else b
    K = b.K if half else bt.shape[1]
    if half and b_self is None:
        if a.n_rows != a.n_cols:
            raise ShapeError("gat_sddmm_aggregate: fp16 rows need fp32 source rows b_self")
        raise ShapeError("gat_sddmm_aggregate: fp16 rows need the fp32 rows as b_self")
    if bt.shape[0] != a.n_cols:
        raise ShapeError("gat_sddmm_aggregate: one B row per column of the pattern required")
    if b_self is None and a.n_rows != a.n_cols:
        raise ShapeError("gat_sddmm_aggregate: a rectangular pattern needs b_self")
    if b_self is not None and (tuple(b_self.shape) != (a.n_rows, K) or b_self.stride(1) != 1):
        raise ShapeError("gat_sddmm_aggregate: b_self must be a row-major n_rows x K tensor")
    if (K > 1024 or K % 4 or _ld(bt) % 4 or bt.data_ptr() % 16 or a_src.data_ptr() % 16
            or a_dst.data_ptr() % 16 or (half and (K % 8 or _ld(bt) % 8 or b.chunks > 1))
            or (b_self is not None and (_ld(b_self) % 4 or b_self.data_ptr() % 16))):
        return None
    _require_cuda(a.col_idx, bt, a_src, a_dst)
    if out is None:
        out = torch.empty(a.n_rows, K, dtype=torch.float32, device=dev)
    if _ld(out) % 4 or out.data_ptr() % 16:
        return None
    code, items, n_items, split, n_split, ws = _plan_args(a, K, algo, dev, gat=True)
    lib = nat.load()
    flags = (nat.GC_RELU if relu else 0) | (nat.GC_SPMM_B_F16 | b.sig_flags() if half else 0)

    def launch(cols, extra):
        return lib.gc_gat_sddmm_aggregate_f32(
            a.row_ptr.data_ptr(), cols.data_ptr(), a_src.data_ptr(), a_dst.data_ptr(), float(slope),
            bt.data_ptr(), _ld(bt), _ptr(b_self), 0 if b_self is None else _ld(b_self),
            b.sigma.data_ptr() if half else None, a.n_rows, K,
            out.data_ptr(), _ld(out), flags | extra, code,
            _ptr(items), n_items, _ptr(split), n_split, _ptr(ws), 0 if ws is None else ws.numel() * 4,
            _stream(dev))

    def probe(cols, extra):
        nat.check(launch(cols, extra), "gat_sddmm_aggregate")

    hints, shrink = _variant(a, K, "gatsdh" if half else "gatsd", probe)
    cols = a.hub_tagged_cols(K) if hints else a.col_idx
    extra = (nat.GC_HUB_TAGGED if hints else 0) | nat.GC_SPMM_SHRINK(shrink)
    rc = _timed_call("spmm", dev, lambda: launch(cols, extra))
    nat.check(rc, "gat_sddmm_aggregate")
    return out


class HalfRows:
    """The TF32 class's half-width gather operand (``gc_pack_rows_f16``): fp16
    rows ``xh`` and per-row scales ``sigma`` with sigma[j] * xh[j] = d[j] *
    x[j] to 11 significant bits — TF32's input rounding — so an aggregation
    gathers 2 bytes per feature instead of 4.  Pass it as the dense operand
    of :func:`spmm` / :func:`spmm_unweighted` (``d_col`` is then carried by
    sigma)."""

    __slots__ = ("xh", "sigma", "K")

    def __init__(self, xh: torch.Tensor, sigma: torch.Tensor, K: int):
        self.xh, self.sigma, self.K = xh, sigma, int(K)

    @property
    def chunks(self) -> int:
        """Scales per row: 1, or one per 256-column chunk (sigma is n x c) as
        the GEMM epilogue emits them for K > 256 (gemm_f16rows)."""
        return 1 if self.sigma.dim() == 1 else int(self.sigma.shape[1])

    def sig_flags(self) -> int:
        return nat.GC_SPMM_SIG_CHUNKS(self.chunks) if self.chunks > 1 else 0

    @property
    def shape(self) -> tuple[int, int]:
        return (self.xh.shape[0], self.K)

    @property
    def device(self) -> torch.device:
        return self.xh.device


def pack_rows_f16(x: torch.Tensor, d: torch.Tensor | None = None, proj: torch.Tensor | None = None):
    """x (n x K fp32, device) -> HalfRows of d·x (d optional, per row; folded
    into the rows before the fp16 rounding, so the row scales sigma are
    powers of two).  ``proj`` (p x K, p <= 16): also return the row
    projections x @ proj.T as a [p, n] tensor, computed from the fp32 rows in
    the same pass (the GAT node scores; returns (HalfRows, proj_out))."""
    _require_cuda(x, d, proj)
    if x.dim() != 2 or x.stride(1) != 1:
        raise ShapeError("pack_rows_f16: x must be a row-major 2-D tensor")
    n, K = x.shape
    if d is not None and tuple(d.shape) != (n,):
        raise ShapeError("pack_rows_f16: d must have one entry per row")
    ldh = (K + 7) // 8 * 8  # 16-byte rows for the gather kernel
    xh = torch.empty(n, ldh, dtype=torch.float16, device=x.device)
    sigma = torch.empty(n, dtype=torch.float32, device=x.device)
    if proj is None:
        nat.check(nat.load().gc_pack_rows_f16(x.data_ptr(), _ld(x), n, K, _ptr(d), xh.data_ptr(),
                                              ldh, sigma.data_ptr(), _stream(x.device)),
                  "pack_rows_f16")
        return HalfRows(xh, sigma, K)
    pj = proj.to(torch.float32).contiguous()
    if pj.dim() != 2 or pj.shape[1] != K or pj.shape[0] > 16:
        raise ShapeError("pack_rows_f16: proj must be p x K with p <= 16")
    out = torch.empty(pj.shape[0], n, dtype=torch.float32, device=x.device)
    nat.check(nat.load().gc_pack_rows_f16_proj(x.data_ptr(), _ld(x), n, K, _ptr(d), xh.data_ptr(),
                                               ldh, sigma.data_ptr(), pj.data_ptr(), pj.shape[0],
                                               out.data_ptr(), _stream(x.device)),
              "pack_rows_f16_proj")
    return HalfRows(xh, sigma, K), out


def _spmm(a: CsrMatrix, b, *, weighted: bool, d_row=None, d_col=None, relu=False, out=None,
          accumulate=False, algo: str = "auto", what="spmm", timer: str | None = "spmm"):
    dev = a.device
    half = isinstance(b, HalfRows)
    if half:
        if d_col is not None:
            raise ShapeError(f"{what}: an fp16 operand carries d_col in its row scales")
        op, bt, d_col = None, b.xh, b.sigma
    else:
        op = _Operand(b, dev)
        bt = op.t
    if a.n_cols != bt.shape[0]:
        raise ShapeError(f"{what}: a is {a.n_rows}x{a.n_cols}, b has {bt.shape[0]} rows")
    K = b.K if half else bt.shape[1]
    _require_cuda(a.col_idx, bt)
    if out is None:
        out = torch.empty(a.n_rows, K, dtype=torch.float32, device=dev)
        if accumulate:
            out.zero_()
    elif tuple(out.shape) != (a.n_rows, K) or out.stride(1) != 1:
        raise ShapeError(f"{what}: out must be a row-major {a.n_rows}x{K} tensor")
    for d, n, nm in ((d_row, a.n_rows, "d_row"), (None if half else d_col, a.n_cols, "d_col")):
        if d is not None and tuple(d.shape) != (n,):
            raise ShapeError(f"{what}: {nm} must have {n} entries")
    if half and d_col.shape[0] != a.n_cols:  # (the fp16 rows' scales: n_cols [x chunks])
        raise ShapeError(f"{what}: the fp16 rows' scales must have {a.n_cols} rows")
    flags = (nat.GC_RELU if relu else 0) | (nat.GC_ACCUMULATE if accumulate else 0) | \
        (nat.GC_SPMM_B_F16 | b.sig_flags() if half else 0)
    code, items, n_items, split, n_split, ws = _plan_args(a, K, algo, dev)
    lib = nat.load()

    def launch(cols, extra, dst=out, fl=flags):
        return lib.gc_spmm_f32(
            a.row_ptr.data_ptr(), cols.data_ptr(), a.values.data_ptr() if weighted else None,
            _ptr(d_row), _ptr(d_col), bt.data_ptr(), _ld(bt), a.n_rows, a.n_cols, K, dst.data_ptr(),
            _ld(dst), fl | extra, code, _ptr(items), n_items, _ptr(split), n_split, _ptr(ws),
            0 if ws is None else ws.numel() * 4, _stream(dev))

    scratch = None

    def probe(cols, extra):
        nonlocal scratch
        if scratch is None:
            scratch = torch.empty(a.n_rows, K, dtype=torch.float32, device=dev)
        nat.check(launch(cols, extra, scratch, flags & ~nat.GC_ACCUMULATE), what)

    hints, shrink = _variant(a, K, "spmmh" if half else "spmm", probe)
    cols = a.hub_tagged_cols(K) if hints else a.col_idx
    extra = (nat.GC_HUB_TAGGED if hints else 0) | nat.GC_SPMM_SHRINK(shrink)
    rc = _timed_call(timer, dev, lambda: launch(cols, extra)) if timer else launch(cols, extra)
    nat.check(rc, what)
    return out if half else op.wrap(out)


def gat_aggregate(a: CsrMatrix, s: torch.Tensor, t: torch.Tensor, slope: float, b, *,
                  relu: bool = False, out=None, algo: str = "auto"):
    """Fused GAT aggregation: C = epi(softmax_row(LeakyReLU(s_i + t_j)) B) with
    the softmax computed online inside the SpMM (α never written) —
    gat.py:72-95 followed by spmm(α, B) (gat.py:127-143) in one kernel."""
    dev = a.device
    half = isinstance(b, HalfRows)
    op = None if half else _Operand(b, dev)
    bt = b.xh if half else op.t
    if a.n_cols != bt.shape[0]:
        raise ShapeError(f"gat_aggregate: a is {a.n_rows}x{a.n_cols}, b has {bt.shape[0]} rows")
    if tuple(s.shape) != (a.n_rows,) or tuple(t.shape) != (a.n_cols,):
        raise ShapeError("gat_aggregate: s/t must have one entry per row/column")
    K = b.K if half else bt.shape[1]
    _require_cuda(a.col_idx, bt, s, t)
    if out is None:
        out = torch.empty(a.n_rows, K, dtype=torch.float32, device=dev)
    elif tuple(out.shape) != (a.n_rows, K) or out.stride(1) != 1:
        raise ShapeError(f"gat_aggregate: out must be a row-major {a.n_rows}x{K} tensor")
    code, items, n_items, split, n_split, ws = _plan_args(a, K, algo, dev, gat=True)
    lib = nat.load()
    flags = (nat.GC_RELU if relu else 0) | (nat.GC_SPMM_B_F16 | b.sig_flags() if half else 0)

    def launch(cols, extra, dst=out):
        return lib.gc_gat_aggregate_f32(
            a.row_ptr.data_ptr(), cols.data_ptr(), s.data_ptr(), t.data_ptr(), float(slope),
            bt.data_ptr(), _ld(bt), b.sigma.data_ptr() if half else None, a.n_rows, a.n_cols, K,
            dst.data_ptr(), _ld(dst), flags | extra,
            code, _ptr(items), n_items, _ptr(split), n_split, _ptr(ws),
            0 if ws is None else ws.numel() * 4, _stream(dev))

    def probe(cols, extra):
        nat.check(launch(cols, extra), "gat_aggregate")  # writes `out`; the real launch follows

    hints, shrink = _variant(a, K, "gath" if half else "gat", probe)
    cols = a.hub_tagged_cols(K) if hints else a.col_idx
    extra = (nat.GC_HUB_TAGGED if hints else 0) | nat.GC_SPMM_SHRINK(shrink)
    rc = _timed_call("spmm", dev, lambda: launch(cols, extra))
    nat.check(rc, "gat_aggregate")
    return out if half else op.wrap(out)


def device_hook(fn):
    """Mark an ``spmm_fn`` hook as device-aware: it receives this package's
    device ``CsrMatrix`` and CUDA operands.  Unmarked hooks get the
    reference's host contract (:func:`call_spmm_hook`)."""
    fn.__gnnc_device__ = True
    return fn


class HostCsrView:
    """Host copy of a CSR with the reference ``CsrMatrix`` attributes
    (``n_rows``, ``n_cols``, int64 ``row_ptr``/``col_idx``, float64
    ``values``, ``nnz``, ``has_unit_values``) — what a reference-style hook
    such as ``gnncompose.sparse.spmm`` (sparse.py:240-247) reads."""

    def __init__(self, a: CsrMatrix):
        self.n_rows, self.n_cols = a.n_rows, a.n_cols
        self.row_ptr, self.col_idx, self.values = a.numpy()
        self.has_unit_values = a.has_unit_values

    @property
    def nnz(self) -> int:
        return int(self.col_idx.size)


def call_spmm_hook(fn, a: CsrMatrix, b):
    """Run a user ``spmm_fn(a, b)`` (reference gcn.py:125-161, gat.py:121-153).
    Device-aware hooks (:func:`device_hook`; this package's ``spmm`` and
    ``spmm_unweighted``) get the device operands.  Any other hook gets the
    reference's host contract — a :class:`HostCsrView` and a float64 ndarray —
    and its ndarray result is uploaded as float32."""
    if getattr(fn, "__gnnc_device__", False):
        out = fn(a, b)
    else:
        bh = b.detach().cpu().numpy().astype(np.float64) if isinstance(b, torch.Tensor) else \
            np.asarray(b, dtype=np.float64)
        out = fn(HostCsrView(a), bh)
    if not isinstance(out, torch.Tensor):
        out = torch.from_numpy(np.ascontiguousarray(out, dtype=np.float32))
    return out.to(a.device, torch.float32)


@device_hook
def spmm(a: CsrMatrix, b, **kw):
    """Sparse-times-dense product C[i,k] = sum_j a[i,j] * b[j,k] (sparse.py:240-247).

    Keyword extensions: ``d_row``/``d_col`` (fused D^-1/2 scalings), ``relu``,
    ``out``, ``accumulate``, ``algo`` in {"auto", "row", "split"}."""
    return _spmm(a, b, weighted=True, what="spmm", **kw)


@device_hook
def spmm_unweighted(a: CsrMatrix, b, **kw):
    """SpMM over the pattern only; ``a.values`` is never read (sparse.py:250-264).
    Bit-identical to ``spmm`` with unit values (same per-row order)."""
    return _spmm(a, b, weighted=False, what="spmm_unweighted", **kw)


def spmm_gemm(a: CsrMatrix, b: torch.Tensor, w: torch.Tensor, *, weighted: bool = True,
              d_row=None, d_col=None, relu: bool = False) -> torch.Tensor:
    """epi(D_row A D_col B) W in one kernel (gc_spmm_gemm_f32): the
    aggregate-first layer's update fused into the SpMM epilogue for a narrow
    W (K1 <= 256, K1 % 4 == 0, K2 <= 32) — reference gcn.py:119-122's
    ``gemm(spmm(a, h), w)`` without the n x K1 round trip.  ``weighted``:
    read ``a.values`` (else unit weights)."""
    _require_cuda(a.col_idx, b, w, d_row, d_col)
    if b.dim() != 2 or b.shape[0] != a.n_cols or b.stride(1) != 1:
        raise ShapeError("spmm_gemm: b must be a row-major n_cols x K1 tensor")
    K1, K2 = b.shape[1], w.shape[1]
    if tuple(w.shape) != (K1, K2):
        raise ShapeError(f"spmm_gemm: w must be {K1} x k2")
    wt = w.to(torch.float32).contiguous()
    out = torch.empty(a.n_rows, K2, dtype=torch.float32, device=b.device)
    nat.check(nat.load().gc_spmm_gemm_f32(
        a.row_ptr.data_ptr(), a.col_idx.data_ptr(), _ptr(a.values) if weighted else None,
        _ptr(d_row), _ptr(d_col), b.data_ptr(), _ld(b), a.n_rows, a.n_cols, K1, wt.data_ptr(), K2,
        out.data_ptr(), K2, nat.GC_RELU if relu else 0, _stream(b.device)), "spmm_gemm")
    return out


def spmm_gemm_eligible(a: CsrMatrix, b, k2: int) -> bool:
    """Shapes the fused aggregate-then-update kernel takes: fp32 rows
    (K1 <= 256, K1 % 4 == 0, 16-byte rows), k2 <= 32, and rows short enough
    for one lane group each (max degree <= SPMM_GEMM_MAX_DEG: the kernel has
    no heavy-row splitting; power-law graphs keep the two-kernel form)."""
    return (SPMM_GEMM and isinstance(b, torch.Tensor) and b.is_cuda and b.dim() == 2
            and b.dtype == torch.float32 and b.stride(1) == 1 and b.shape[1] % 4 == 0
            and _ld(b) % 4 == 0 and b.data_ptr() % 16 == 0 and 0 < b.shape[1] <= 256
            and 0 < k2 <= 32 and a.max_degree() <= SPMM_GEMM_MAX_DEG)


# ---------------------------------------------------------------------------
# SDDMM — reference sparse.py:267-282
# ---------------------------------------------------------------------------


def sddmm(a: CsrMatrix, b, c) -> CsrMatrix:
    """Masked product d[i,j] = a[i,j] * sum_k b[i,k] c[j,k]; the output shares
    a's pattern."""
    dev = a.device
    bt, ct = _Operand(b, dev).t, _Operand(c, dev).t
    if bt.shape[0] != a.n_rows:
        raise ShapeError(f"sddmm: b has {bt.shape[0]} rows, expected {a.n_rows}")
    if ct.shape[0] != a.n_cols:
        raise ShapeError(f"sddmm: c has {ct.shape[0]} rows, expected {a.n_cols}")
    if bt.shape[1] != ct.shape[1]:
        raise ShapeError("sddmm: b and c must have the same column count")
    _require_cuda(a.col_idx, bt, ct)
    out = torch.empty(a.nnz, dtype=torch.float32, device=dev)
    if a.nnz:
        nat.check(nat.load().gc_sddmm_f32(a.row_ptr.data_ptr(), a.col_idx.data_ptr(),
                                          a.values.data_ptr(), bt.data_ptr(), _ld(bt), ct.data_ptr(),
                                          _ld(ct), a.n_rows, a.n_cols, bt.shape[1], out.data_ptr(),
                                          _stream(dev)), "sddmm")
    return a.with_values(out)


def sddmm_norm(a: CsrMatrix, d: torch.Tensor, *, weighted: bool = True) -> CsrMatrix:
    """k = 1 SDDMM a[i,j] * (d[i] * d[j]) — the normalised adjacency of
    gcn.py:103-112 in one pass."""
    dev = _require_cuda(a.col_idx, d)
    if tuple(d.shape) != (a.n_rows,) or a.n_rows != a.n_cols:
        raise ShapeError("degree vector does not match the adjacency")
    out = torch.empty(a.nnz, dtype=torch.float32, device=dev)
    if a.nnz:
        nat.check(nat.load().gc_sddmm_norm_f32(a.row_ptr.data_ptr(), a.col_idx.data_ptr(),
                                               a.values.data_ptr() if weighted else None,
                                               d.data_ptr(), a.n_rows, a.nnz, out.data_ptr(),
                                               _stream(dev)), "sddmm_norm")
    return a.with_values(out)


# ---------------------------------------------------------------------------
# dense — reference sparse.py:285-300
# ---------------------------------------------------------------------------

_GEMM_PRECISION = os.environ.get("GNNC_GEMM_PRECISION", "tf32")


def set_gemm_precision(p: str) -> None:
    """The numerics class of the dense update (and of the dense split's
    operand terms, hub.py):

    * "tf32" — one tcgen05 kind::tf32 MMA per product (TF32 input rounding,
      fp32 accumulation); parity class 1e-2;
    * "fp32" — 3xTF32 on tcgen05 (hi·hi + hi·lo + lo·hi, the fp32 operands
      split into TF32 hi/lo terms on chip); parity class 1e-4.  Operands TMA
      cannot describe (row pitch not a multiple of 16 bytes) take the exact
      CUDA-core kernel."""
    global _GEMM_PRECISION
    if p not in ("tf32", "fp32"):
        raise ValueError("precision must be 'tf32' or 'fp32'")
    _GEMM_PRECISION = p


def get_gemm_precision() -> str:
    return _GEMM_PRECISION


def gemm(a, b, *, row_scale=None, relu=False, precision: str | None = None, out=None):
    """Dense product a @ b (sparse.py:285-291) on the tcgen05 tensor cores
    (TF32, or 3xTF32 in the fp32 class); ``precision="simt"`` forces the
    exact-fp32 CUDA-core kernel.  Optional fused row scale and ReLU."""
    dev = b.device if isinstance(b, torch.Tensor) else (
        a.device if isinstance(a, torch.Tensor) else default_device())
    oa, ob = _Operand(a, dev), _Operand(b, dev)
    at, bt = oa.t, ob.t
    if at.shape[1] != bt.shape[0]:
        raise ShapeError(f"gemm: inner dimensions {at.shape[1]} != {bt.shape[0]}")
    _require_cuda(at, bt, row_scale)
    M, K, N = at.shape[0], at.shape[1], bt.shape[1]
    if out is None:
        out = torch.empty(M, N, dtype=torch.float32, device=dev)
    prec = precision or _GEMM_PRECISION
    if prec not in ("tf32", "fp32", "simt"):
        raise ValueError("precision must be 'tf32', 'fp32' or 'simt'")
    flags = nat.GC_RELU if relu else 0
    lib = nat.load()
    ws = None
    tensor = prec in ("tf32", "fp32")
    if tensor and K >= 8 and (_ld(at) % 4 or at.data_ptr() % 16) and M * K <= (1 << 28):
        # TMA needs 16-byte row pitch: stage A with a padded leading dimension
        # (e.g. Cora's k1 = 1433 -> 1436) through the row-copy kernel
        ldp = (K + 3) // 4 * 4
        ap = torch.empty(M, ldp, dtype=torch.float32, device=dev)
        nat.check(lib.gc_scale_rows_f32(None, at.data_ptr(), _ld(at), M, K, ap.data_ptr(), ldp, 0,
                                        _stream(dev)), "gemm(pad)")
        at = ap[:, :K]
    if tensor and (_ld(at) % 4 == 0) and at.data_ptr() % 16 == 0 and K > 0:
        flags |= nat.GC_GEMM_TF32 if prec == "tf32" else nat.GC_GEMM_TF32X3
        ws = torch.empty(max(int(lib.gc_gemm_workspace_bytes(K, N)), 16), dtype=torch.uint8,
                         device=dev)
    else:
        flags |= nat.GC_GEMM_FP32
    if row_scale is not None and tuple(row_scale.shape) != (M,):
        raise ShapeError("gemm: row_scale must have one entry per row")
    rc = _timed_call("gemm", dev, lambda: lib.gc_gemm_f32(
        at.data_ptr(), _ld(at), bt.data_ptr(), _ld(bt), M, K, N, out.data_ptr(), _ld(out),
        _ptr(row_scale), flags, _ptr(ws), 0 if ws is None else ws.numel(), _stream(dev)))
    nat.check(rc, "gemm")
    return oa.wrap(out) if (oa.host and ob.host) else out


def gemm_f16rows(a: torch.Tensor, b: torch.Tensor, *, row_scale=None) -> HalfRows | None:
    """(diag(row_scale) a @ b) produced directly as the TF32 class's fp16
    gather operand (``HalfRows``) by the TF32 tcgen05 GEMM's epilogue — the
    fp32 product is never written.  None when the shape is outside the fused
    epilogue's range (N > 256, unaligned A): the caller then packs."""
    _require_cuda(a, b, row_scale)
    M, K = a.shape
    N = b.shape[1]
    if b.shape[0] != K:
        raise ShapeError(f"gemm: inner dimensions {K} != {b.shape[0]}")
    if (N > 256 and (N % 256 or not F16ROWS_CHUNKED)) or K < 1 or a.stride(1) != 1 \
            or _ld(a) % 4 or a.data_ptr() % 16:
        return None
    if row_scale is not None and tuple(row_scale.shape) != (M,):
        raise ShapeError("gemm: row_scale must have one entry per row")
    bt = b.contiguous() if b.stride(1) != 1 else b
    lib = nat.load()
    ldh = (N + 7) // 8 * 8
    xh = torch.empty(M, ldh, dtype=torch.float16, device=a.device)
    # one scale per row, or per row and 256-column chunk (N > 256)
    sigma = torch.empty((M,) if N <= 256 else (M, N // 256), dtype=torch.float32, device=a.device)
    ws = torch.empty(max(int(lib.gc_gemm_workspace_bytes(K, N)), 16), dtype=torch.uint8,
                     device=a.device)
    rc = _timed_call("gemm", a.device, lambda: lib.gc_gemm_f16rows_f32(
        a.data_ptr(), _ld(a), bt.data_ptr(), _ld(bt), M, K, N, _ptr(row_scale), xh.data_ptr(), ldh,
        sigma.data_ptr(), ws.data_ptr(), ws.numel(), _stream(a.device)))
    nat.check(rc, "gemm_f16rows")
    return HalfRows(xh, sigma, N)


def scale_rows(d, b, *, relu: bool = False):
    """Row scaling out[i,k] = d[i] * b[i,k] (sparse.py:294-300)."""
    dev = b.device if isinstance(b, torch.Tensor) else default_device()
    ob = _Operand(b, dev)
    bt = ob.t
    dt = d if isinstance(d, torch.Tensor) else torch.as_tensor(np.asarray(d, dtype=np.float64))
    dt = dt.to(dev, torch.float32).contiguous()
    if dt.dim() != 1 or dt.numel() != bt.shape[0]:
        raise ShapeError(f"scale_rows: d has {dt.numel()} entries, b has {bt.shape[0]} rows")
    _require_cuda(bt, dt)
    out = torch.empty_like(bt)
    nat.check(nat.load().gc_scale_rows_f32(dt.data_ptr(), bt.data_ptr(), _ld(bt), bt.shape[0],
                                           bt.shape[1], out.data_ptr(), _ld(out),
                                           nat.GC_RELU if relu else 0, _stream(dev)), "scale_rows")
    return ob.wrap(out)


def relu_(x: torch.Tensor) -> torch.Tensor:
    """In-place ReLU through the kernel library (gcn.py:115-116)."""
    dev = _require_cuda(x)
    nat.check(nat.load().gc_scale_rows_f32(None, x.data_ptr(), _ld(x), x.shape[0], x.shape[1],
                                           x.data_ptr(), _ld(x), nat.GC_RELU, _stream(dev)), "relu")
    return x


# ---------------------------------------------------------------------------
# graph prep — reference sparse.py:303-336
# ---------------------------------------------------------------------------


def add_self_loops(a: CsrMatrix) -> CsrMatrix:
    """Insert value-1.0 diagonal entries where absent; existing ones are kept.
    Idempotent.  O(nnz) insertion into the sorted CSR (no re-sort); the
    result is bit-identical to the reference's from_coo rebuild."""
    if a.n_rows != a.n_cols:
        raise ShapeError("add_self_loops requires a square matrix")
    dev = a.device
    n = a.n_rows
    rows = a.row_of_nnz()
    col = a.col_idx.long()
    has_diag = torch.zeros(n, dtype=torch.bool, device=dev)
    has_diag[rows[col == rows]] = True
    missing = ~has_diag
    n_missing = int(missing.sum())
    if n_missing == 0:
        return a
    deg = a.degrees()
    new_deg = deg + missing.long()
    row_ptr = torch.cat([new_deg.new_zeros(1), torch.cumsum(new_deg, 0)])
    shift = torch.cumsum(missing.long(), 0) - missing.long()  # missing rows before r
    after_diag = (missing[rows] & (col > rows)).long()
    new_pos = torch.arange(a.nnz, device=dev) + shift[rows] + after_diag
    lt = torch.zeros(n, dtype=torch.long, device=dev)
    lt.index_add_(0, rows, (col < rows).long())  # integer adds: exact, order-free
    miss_rows = torch.nonzero(missing).reshape(-1)
    diag_pos = row_ptr[miss_rows] + lt[miss_rows]
    m2 = a.nnz + n_missing
    new_col = torch.empty(m2, dtype=torch.int32, device=dev)
    new_val = torch.empty(m2, dtype=torch.float32, device=dev)
    new_col[new_pos] = a.col_idx
    new_val[new_pos] = a.values
    new_col[diag_pos] = miss_rows.to(torch.int32)
    new_val[diag_pos] = 1.0
    out = CsrMatrix(n, n, row_ptr, new_col, new_val, validate=False, device=dev)
    if a._unit:
        out._unit = True
    return out


def inv_sqrt_degrees(a: CsrMatrix) -> torch.Tensor:
    """d_i = (structural degree)^-1/2 (sparse.py:327-336), computed in float64
    and rounded once to float32."""
    deg = a.degrees()
    if a.n_rows and bool((deg == 0).any()):
        bad = int(torch.nonzero(deg == 0)[0])
        raise DegenerateNodeError(f"node {bad} has zero degree; add self loops first")
    return (1.0 / torch.sqrt(deg.double())).float()
