"""Hybrid aggregation for power-law graphs: dense blocks of the adjacency on
the tensor cores, the sparse remainder on the SpMM kernel.

On a dense power-law graph (Reddit-shaped: mean degree ~490) the SpMM is
bound by L2 bandwidth, not HBM: every edge gathers a K-wide row of X and the
most-referenced columns are gathered again and again.  Ordering rows and
columns by degree exposes dense regions of

    C = D Ã D X          (the reference's dynamic form, gcn.py:137-155;
                          precompute's Ñ = D Ã D, gcn.py:103-112)

that are cheaper as dense products whose operand tiles are reused from
shared memory:

    C_dense = D · A_dense · (D X)[dense columns],   A_dense ∈ {0,1}

computed by tcgen05 kind::f16 GEMMs: the 0/1 blocks are exact in fp16/bf16
and (D X)[columns] is rounded to 16-bit terms (``gc_hub_pack``) following
the layer's GEMM precision (``sparse.set_gemm_precision``): in the TF32 mode
(1e-2 parity, the default) one fp16 term of s·D·X with a power-of-two scale
s — 11 significant bits, the same input rounding the TF32 update GEMM
applies to H; in the fp32 mode (1e-4 parity) two fp16 terms (22 significant
bits: absolute error <= 2^-23·max|D X| per element).  GNNC_HUB_FORMAT pins
"f16", "f16x2" or "bf16x3" (three bf16 terms carrying the exact fp32
mantissa).  The SpMM then accumulates the remaining edges on top
(GC_ACCUMULATE); apart from the term split only the summation order differs
from the plain SpMM.

Two plans:

* ``HubPlan`` (block, T): every row against the T most-referenced columns
  (one dense n × T block; supports row ranges, any K).
* ``StairPlan`` ("stair", δ): rows and columns in degree-rank order; step s
  is the block rows [0, R_s) × columns [C_s, C_{s+1}) with R_s the last row
  band whose density in that column band is ≥ δ — a staircase hugging the
  dense corner (the high-degree rows are dense far beyond the top columns).
  All steps run in ONE CTA-pair GEMM whose rank-ordered tiles reduce over a
  prefix of the steps (``gc_hub_stair_gemm``), scattering rows back
  through the rank permutation.

The split applies to a unit-valued Ã (the reference's own generated graphs and
``has_unit_values`` case); the plan is chosen per (pattern, K) by timing the
candidates once, like the SpMM variant autotuner (reference tiling.py:311-364
is the CPU analogue).  GNNC_HUB_SPLIT: "auto" (default), "0" (off), "<T>"
(block plan), "stair:<δ in permille>".
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native as nat
from .sparse import (CsrMatrix, HalfRows, ShapeError, _ld, _ptr, _require_cuda, _spmm, _stream,
                     _timed_call)

HUB_SPLIT = os.environ.get("GNNC_HUB_SPLIT", "auto")
# term format of the dense operand: "auto" (default: one fp16 term in the TF32
# GEMM mode, two in the fp32 mode), "f16" (one fp16 term of s·D·X, 11
# significant bits), "f16x2" (two fp16 terms — 22 significant bits, absolute
# error <= 2^-23 max|D·X| per element, 2/3 of the MMAs of bf16x3; Reddit K=256
# staircase 0.58 vs 0.80 ms, normwise difference from the plain SpMM 2.8e-6
# either way) or "bf16x3" (exact fp32 split)
HUB_FORMAT = os.environ.get("GNNC_HUB_FORMAT", "auto")
_TERMS = {nat.GC_HUB_F16: 1, nat.GC_HUB_F16_MN: 1, nat.GC_HUB_F16X2: 2, nat.GC_HUB_BF16X3: 3}
FORMAT_NAMES = {nat.GC_HUB_F16: "f16", nat.GC_HUB_F16_MN: "f16", nat.GC_HUB_F16X2: "f16x2",
                nat.GC_HUB_BF16X3: "bf16x3"}


def _fmt() -> int:
    """The 0/1 block family of a plan: bf16 blocks for bf16x3, else fp16."""
    return nat.GC_HUB_BF16X3 if HUB_FORMAT == "bf16x3" else nat.GC_HUB_F16X2


def term_format(block_fmt: int | None = None) -> int:
    """The term format a pack/GEMM runs in now (see HUB_FORMAT)."""
    if (block_fmt if block_fmt is not None else _fmt()) == nat.GC_HUB_BF16X3:
        return nat.GC_HUB_BF16X3
    if HUB_FORMAT == "f16":
        return nat.GC_HUB_F16
    if HUB_FORMAT == "f16x2":
        return nat.GC_HUB_F16X2
    from .sparse import get_gemm_precision

    return nat.GC_HUB_F16 if get_gemm_precision() == "tf32" else nat.GC_HUB_F16X2


def term_count(fmt: int | None = None) -> int:
    return _TERMS[term_format() if fmt is None else fmt]


def _block_dtype(fmt: int):
    return torch.bfloat16 if fmt == nat.GC_HUB_BF16X3 else torch.float16
# staircase blocks as bitmaps (GC_HUB_A_BITS: converter warps expand them in
# shared memory; 1/16 of the 16-bit blocks' HBM footprint).  Off by default:
# measured 0.86 vs 0.62 ms on Reddit K=256 — handoff-latency bound (gemm.cu)
HUB_ABITS = os.environ.get("GNNC_HUB_ABITS", "0") == "1"
# (cell/edge cost ratio δ, balance slack) pairs tried by the autotuner
# (slack > 1 reaches further right, but short-wide steps stream their B
# operand from DRAM once per pair tile and lose to the tail: measured 2.73 ms
# at (0.012, 1.0) vs 2.99 ms at (0.018, 3.0) on Reddit K=256)
STAIR_CANDIDATES = ((0.008, 1.0), (0.012, 1.0), (0.018, 1.0))
# narrower feature rows make a dense cell relatively dearer (the tensor tile
# is N = K wide: A-operand bound), so small K tries sparser staircases
STAIR_CANDIDATES_SMALL_K = {128: ((0.018, 1.0), (0.03, 1.0), (0.06, 1.0)),
                            64: ((0.03, 1.0), (0.06, 1.0), (0.12, 1.0)),
                            32: ((0.03, 1.0), (0.06, 1.0), (0.12, 1.0))}


def _stair_candidates(K: int):
    """δ candidates for this K, tuned on the two-term format; a dense cell
    costs MMAs in proportion to the term count, so δ scales with it (the
    one-term format also keeps the two-term table's two smallest δ: with
    fp16 tail rows the tail is cheaper, so sparser staircases can win)."""
    cands = STAIR_CANDIDATES
    for k, c in sorted(STAIR_CANDIDATES_SMALL_K.items()):
        if K <= k:
            cands = c
            break
    f = term_count() / 2.0
    if f == 1.0:
        return cands
    out = [(max(round(dl * f, 3), 0.001), sl) for dl, sl in cands]
    if f < 1.0:
        out.extend(cands[:2])
    return tuple(dict.fromkeys(out))
HUB_MIN_NNZ = 1 << 24            # smaller graphs stay on the SpMM alone
HUB_MEM_BUDGET = 8 << 30         # bytes of dense blocks per pattern
STAIR_MAX_STEPS = 16
STAIR_FIRST_BAND = 1024          # rows / columns of the first histogram band
AUTOTUNE_ROUNDS = 7              # interleaved timing rounds per candidate
STAIR_BAND_RATIO = 2 ** 0.5      # growth of the histogram bands
STAIR_CLUSTERS = 74              # CTA pairs of a B200 (balance bound of the top tile)


def _unit_tail(a: CsrMatrix, keep: torch.Tensor, rows: torch.Tensor) -> CsrMatrix:
    cnt = torch.bincount(rows[keep], minlength=a.n_rows)
    rp = torch.zeros(a.n_rows + 1, dtype=torch.int32, device=a.device)
    rp[1:] = torch.cumsum(cnt, 0).to(torch.int32)
    tail = CsrMatrix(a.n_rows, a.n_cols, rp, a.col_idx[keep].contiguous(),
                     torch.ones(keep.numel(), dtype=torch.float32, device=a.device),
                     validate=False, device=a.device)
    tail._unit = True
    return tail


class _TailMixin:
    """The remainder pattern and its row blocks, carrying unit values or a
    same-pattern matrix's values (e.g. Ñ's) gathered at the tail positions."""

    def _init_tail(self, a: CsrMatrix, keep_mask: torch.Tensor, rows: torch.Tensor):
        keep = torch.nonzero(keep_mask).flatten()
        self.keep = keep
        self.tail = _unit_tail(a, keep, rows)
        self.hub_edges = a.nnz - keep.numel()
        self._tail_vals: dict = {}

    def tail_block(self, values: torch.Tensor | None, lo: int, hi: int) -> CsrMatrix:
        # keyed on the values tensor itself (held, so its id cannot be reused
        # by a new tensor) and its version (in-place updates invalidate)
        vkey = None if values is None else (id(values), values._version)
        hit = self._tail_vals.get(vkey)
        if hit is None or (values is not None and hit[0] is not values):
            self._tail_vals = {k: v for k, v in self._tail_vals.items() if k is None}
            hit = (values, {}, self.tail if values is None
                   else self.tail.with_values(values[self.keep].contiguous()))
            self._tail_vals[vkey] = hit
        _, blocks, full = hit
        if (lo, hi) == (0, full.n_rows):
            return full
        if (lo, hi) not in blocks:
            blocks[(lo, hi)] = full.take_rows(lo, hi)
            blocks[(lo, hi)]._unit = values is None
        return blocks[(lo, hi)]


class HubPlan(_TailMixin):
    """Column split of one pattern: hub columns, the dense 0/1 hub block
    (bf16, row-major n × T) and the tail pattern (CSR without the hub
    columns; ``keep`` maps tail positions back to the full pattern)."""

    kind = "block"

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
        self.fmt = _fmt()
        self.hub_cols = hub.to(torch.int32).contiguous()
        self.a_hub = torch.zeros(a.n_rows, T, dtype=_block_dtype(self.fmt), device=dev)
        self.a_hub[rows[is_hub], colpos[is_hub]] = 1.0
        self.cells = a.n_rows * T
        self._init_tail(a, ~is_hub, rows)


class StairPlan(_TailMixin):
    """Degree-rank staircase of dense blocks (see the module docstring)."""

    kind = "stair"

    def __init__(self, a: CsrMatrix, delta: float, *, slack: float = 1.0,
                 n_clusters: int = STAIR_CLUSTERS, first_band: int = 1024):
        dev = a.device
        col = a.col_idx.long()
        ccount = torch.bincount(col, minlength=a.n_cols)
        corder = torch.argsort(ccount, descending=True, stable=True)
        crank = torch.empty_like(corder)
        crank[corder] = torch.arange(a.n_cols, device=dev)
        rdeg = a.degrees()
        rorder = torch.argsort(rdeg, descending=True, stable=True)
        rrank = torch.empty_like(rorder)
        rrank[rorder] = torch.arange(a.n_rows, device=dev)
        rows = a.row_of_nnz()
        er, ec = rrank[rows], crank[col]
        self.steps = self._staircase(a, er, ec, delta, slack, n_clusters, first_band)
        if not self.steps:
            raise ValueError("stair split: no block pays for its cells")
        cells = sum(R * W for R, _, W in self.steps)
        if cells * (0.125 if HUB_ABITS else 2) > HUB_MEM_BUDGET:
            # checked before any block is allocated
            raise ValueError(f"stair split: {cells} cells exceed the dense-block budget")
        C = self.steps[-1][1] + self.steps[-1][2]
        self.T = C
        self.delta = delta
        self.hub_cols = corder[:C].to(torch.int32).contiguous()
        self.row_map = rorder.to(torch.int32).contiguous()
        self.rows0 = self.steps[0][0]
        # step of each covered edge: column rank band, then the row limit
        c_starts = torch.tensor([s[1] for s in self.steps], device=dev)
        r_limits = torch.tensor([s[0] for s in self.steps], device=dev)
        in_cols = ec < C
        step = torch.bucketize(ec.clamp(max=C - 1), c_starts, right=True) - 1
        covered = in_cols & (er < r_limits[step])
        self.blocks = []
        self.fmt = _fmt()
        self.abits = HUB_ABITS
        for s, (R, c0, W) in enumerate(self.steps):
            sel = covered & (step == s)
            if self.abits:
                # word (k, r) at k * rpad + r; the edges of a row are distinct
                # columns, so summing their bits is OR-ing them
                rpad = -(-R // 256) * 256
                c = ec[sel] - c0
                blk = torch.zeros((W // 64) * rpad, dtype=torch.int64, device=dev)
                blk.index_add_(0, (c // 64) * rpad + er[sel],
                               torch.bitwise_left_shift(torch.ones_like(c), c % 64))
            else:
                blk = torch.zeros(R, W, dtype=_block_dtype(self.fmt), device=dev)
                blk[er[sel], ec[sel] - c0] = 1.0
            self.blocks.append(blk)
        self.cells = sum(R * W for R, _, W in self.steps)
        self._np_rows = np.array([s[0] for s in self.steps], np.int64)
        self._np_c0 = np.array([s[1] for s in self.steps], np.int64)
        self._np_w = np.array([s[2] for s in self.steps], np.int64)
        self._np_ptrs = np.array([b.data_ptr() for b in self.blocks], np.uint64)
        self._sched: dict = {}
        self._init_tail(a, ~covered, rows)

    def dense_block(self, s: int) -> torch.Tensor:
        """Step s's 0/1 block as a float [R x W] tensor (either storage)."""
        R, _, W = self.steps[s]
        blk = self.blocks[s]
        if not self.abits:
            return blk.float()
        rpad = -(-R // 256) * 256
        words = blk.view(W // 64, rpad)
        j = torch.arange(64, device=blk.device)
        bits = (words.unsqueeze(-1) >> j) & 1  # [k, r, 64]
        return bits.permute(1, 0, 2).reshape(rpad, W)[:R].float()

    def schedule(self, K: int, device):
        """Work items for the staircase GEMM, longest-processing-time first
        over the CTA pairs.  Pair tiles (256 rank-ordered rows x one N tile)
        reduce over different step prefixes; a tile longer than the mean
        per-pair load is cut into split-K chunks (the first writes C, the rest
        write workspace slots that a fixup adds in slot order).  Returns
        (items int32[n][4], cluster_start, n_clusters, workspace | None,
        fixups int32[f][4] | None)."""
        if K not in self._sched:
            import heapq

            pbn = int(nat.load().gc_hub_stair_pair_bn(K))
            n_tiles = -(-K // pbn)
            m_pairs = -(-self.rows0 // 256)
            kb = [sum(w // 64 for r, _, w in self.steps if r > mp * 256) for mp in range(m_pairs)]
            sms = torch.cuda.get_device_properties(device).multi_processor_count
            total = sum(kb) * n_tiles
            n_cl = max(1, min(m_pairs * n_tiles, sms // 2))
            target = max(16, -(-total // n_cl))
            items, fixups, slot = [], [], 0
            for mp in range(m_pairs):
                for nt in range(n_tiles):
                    t = mp * n_tiles + nt
                    parts = -(-kb[mp] // target) if kb[mp] > target else 1
                    if parts == 1:
                        items.append((kb[mp], (t, 0, -1, -1)))
                        continue
                    bounds = [kb[mp] * i // parts for i in range(parts + 1)]
                    items.append((bounds[1], (t, 0, bounds[1], -1)))
                    fixups.append((t, slot, parts - 1, 0))
                    for i in range(1, parts):
                        items.append((bounds[i + 1] - bounds[i], (t, bounds[i], bounds[i + 1], slot)))
                        slot += 1
            items.sort(key=lambda x: -x[0])
            heap = [(0, c) for c in range(n_cl)]
            lists: list[list] = [[] for _ in range(n_cl)]
            for w, it in items:
                load, c = heapq.heappop(heap)
                lists[c].append(it)
                heapq.heappush(heap, (load + w + 4, c))  # + per-item epilogue cost
            starts = np.zeros(n_cl + 1, np.int32)
            starts[1:] = np.cumsum([len(x) for x in lists])
            flat = np.array([v for x in lists for it in x for v in it], np.int32)
            ws = torch.empty(max(slot, 1) * 256 * pbn, dtype=torch.float32, device=device) \
                if slot else None
            fx = torch.from_numpy(np.array(fixups, np.int32).reshape(-1, 4)).to(device) \
                if fixups else None
            self._sched[K] = (torch.from_numpy(flat).to(device), torch.from_numpy(starts).to(device),
                              n_cl, ws, fx)
        return self._sched[K]

    @staticmethod
    def _bands(n: int, first: int, align: int) -> list[int]:
        """0, first, then geometric boundaries (STAIR_BAND_RATIO, multiples of
        ``align``), n."""
        b, x = [0], float(first)
        while int(x) // align * align < n:
            v = int(x) // align * align
            if v > b[-1]:
                b.append(v)
            x *= STAIR_BAND_RATIO
        if b[-1] != n:
            b.append(n)
        return b

    @classmethod
    def _staircase(cls, a: CsrMatrix, er, ec, delta, slack, n_clusters,
                   first_band: int = 1024) -> list[tuple[int, int, int]]:
        """[(R_s, C_s, W_s)]: per column band (rank order, multiples of 64),
        the row prefix R maximising edges − δ·cells (δ = cell cost / edge
        cost), never growing from one band to the next; adjacent bands with
        the same R merge into one step (<= STAIR_MAX_STEPS).  Stops when the
        top tile's reduction would exceed slack × the mean per-cluster load."""
        cmax = a.n_cols // 64 * 64
        if cmax < 64:
            return []
        rb = cls._bands(a.n_rows, first_band, 128)
        cb = cls._bands(cmax, first_band, 64)
        dev = er.device
        ri = torch.bucketize(er, torch.tensor(rb[1:-1], device=dev), right=True)
        ci = torch.bucketize(ec, torch.tensor(cb[1:-1], device=dev), right=True)
        valid = ec < cmax
        nr, nc = len(rb) - 1, len(cb) - 1
        H = torch.zeros(nr * nc, dtype=torch.int64, device=dev)
        H.index_add_(0, (ri * nc + ci)[valid], torch.ones_like(ri[valid]))
        H = H.view(nr, nc).cpu().numpy()
        steps: list[list[int]] = []
        prev_r = a.n_rows
        work = 0.0  # pair k-blocks of the bands taken
        for s in range(nc):
            W = cb[s + 1] - cb[s]
            best_r, best_gain, cum = 0, 0.0, 0
            for b in range(nr):
                if rb[b + 1] > prev_r:
                    break
                cum += int(H[b, s])
                gain = cum - delta * rb[b + 1] * W
                if gain > best_gain:
                    best_gain, best_r = gain, rb[b + 1]
            if best_r < first_band:
                break
            w_new = work + best_r * W / (256.0 * 64.0)
            if steps and cb[s + 1] / 64.0 > slack * w_new / n_clusters:
                break  # the top tile would outlast the average cluster
            if steps and steps[-1][0] == best_r:
                steps[-1][2] += W  # same rows: widen the previous step
            elif len(steps) == STAIR_MAX_STEPS:
                break
            else:
                steps.append([best_r, cb[s], W])
            work, prev_r = w_new, best_r
        return [tuple(x) for x in steps]


def _parse_spec(spec):
    """0 | T (block plan) | ("stair", δ permille, slack tenths) |
    "stair:<permille>[:<slack tenths>]" | "<T>"."""
    if isinstance(spec, tuple):
        return spec if len(spec) == 3 else (spec[0], spec[1], 10)
    if isinstance(spec, str) and spec.startswith("stair:"):
        parts = spec.split(":")
        return ("stair", int(parts[1]), int(parts[2]) if len(parts) > 2 else 10)
    return int(spec)


def spec_label(spec) -> str:
    spec = _parse_spec(spec)
    return f"stair:{spec[1]}:{spec[2]}" if isinstance(spec, tuple) else str(spec)


def hub_plan(a: CsrMatrix, spec):
    spec = _parse_spec(spec)
    key = ("hubsplit", spec)
    if key not in a._plans:
        if isinstance(spec, tuple):
            a._plans[key] = StairPlan(a, spec[1] / 1000.0, slack=spec[2] / 10.0,
                                      first_band=STAIR_FIRST_BAND)
        else:
            a._plans[key] = HubPlan(a, spec)
    return a._plans[key]


def pack(a: CsrMatrix, x: torch.Tensor, d: torch.Tensor, spec):
    """The dense-part operand (D X)[hub_cols] as bf16/fp16 terms, K-major,
    the fp16 formats' scale workspace (float[2]: max, 1/s) and the term
    format used (``term_format``)."""
    plan = hub_plan(a, spec)
    lib = nat.load()
    half = isinstance(x, HalfRows)
    K = x.K if half else x.shape[1]
    kp = int(lib.gc_hub_terms_rows(K))
    fmt = term_format(plan.fmt)
    if fmt == nat.GC_HUB_F16 and not getattr(plan, "abits", False) \
            and lib.gc_hub_f16_mn_supported(K):
        fmt = nat.GC_HUB_F16_MN  # rows as gathered: no transpose in the pack
    if half and fmt not in (nat.GC_HUB_F16, nat.GC_HUB_F16_MN):
        raise ShapeError("hub pack: fp16 gather rows carry the one-term (TF32 class) format only")
    bt = torch.empty(_TERMS[fmt] * kp * plan.T, dtype=_block_dtype(fmt), device=x.device)
    sc = torch.empty(2, dtype=torch.float32, device=x.device)
    if half:  # the dense part reads the same fp16 rows as the tail
        fmt_c = fmt | (nat.GC_HUB_SIG_CHUNKS(x.chunks) if x.chunks > 1 else 0)
        nat.check(lib.gc_hub_pack_f16rows(x.xh.data_ptr(), _ld(x.xh), x.sigma.data_ptr(), K,
                                          plan.hub_cols.data_ptr(), plan.T, _ptr(d), fmt_c,
                                          bt.data_ptr(), sc.data_ptr(), _stream(x.device)),
                  "hub_pack_f16rows")
        return bt, sc, fmt
    nat.check(lib.gc_hub_pack(x.data_ptr(), _ld(x), K, plan.hub_cols.data_ptr(), plan.T,
                              None if d is None else d.data_ptr(), fmt, bt.data_ptr(),
                              sc.data_ptr(),
                              _stream(x.device)), "hub_pack")
    return bt, sc, fmt


_SIDE_STREAMS: dict = {}


def dense_part(a: CsrMatrix, x: torch.Tensor, d: torch.Tensor, spec, out: torch.Tensor, *,
               d_row: torch.Tensor, accumulate: bool = False, packed=None,
               rows: tuple[int, int] | None = None) -> None:
    """out (rows [lo, hi) of C, or all of C) = / += D_row · A_dense · (D X)[...]."""
    plan = hub_plan(a, spec)
    dev = x.device
    lib = nat.load()
    st = _stream(dev)
    K = x.K if isinstance(x, HalfRows) else x.shape[1]
    zero_done = None
    if plan.kind == "stair" and plan.rows0 < a.n_rows and not accumulate \
            and (rows is None or tuple(rows) == (0, a.n_rows)):
        # rows outside every step receive only the tail: zero them on a side
        # stream while the operand is packed (independent memory)
        main = torch.cuda.current_stream(dev)
        side = _SIDE_STREAMS.setdefault(dev, torch.cuda.Stream(dev))
        side.wait_stream(main)
        outside = plan.row_map[plan.rows0:]  # original ids of the rows beyond every step
        with torch.cuda.stream(side):
            nat.check(lib.gc_zero_rows(out.data_ptr(), _ld(out), outside.data_ptr(),
                                       outside.numel(), K, _stream(dev)), "zero_rows")
        out.record_stream(side)
        zero_done = torch.cuda.Event()
        zero_done.record(side)
    bt, sc, fmt = packed if packed is not None else pack(a, x, d, spec)
    flags = nat.GC_ACCUMULATE if accumulate else 0
    if plan.kind == "block":
        lo, hi = rows if rows is not None else (0, a.n_rows)
        a_hub = plan.a_hub[lo:hi]
        dr = d_row[lo:hi]
        nat.check(_timed_call("hub_gemm", dev, lambda: lib.gc_hub_gemm(
            a_hub.data_ptr(), plan.T, hi - lo, plan.T, bt.data_ptr(), K, fmt, sc.data_ptr(),
            out.data_ptr(), _ld(out), dr.data_ptr(), flags, st)), "hub_gemm")
        return
    if rows is not None and tuple(rows) != (0, a.n_rows):
        raise ShapeError("stair split: the dense part covers all rows (rank-ordered tiles)")
    if zero_done is not None:
        torch.cuda.current_stream(dev).wait_event(zero_done)
    _stair_gemm(plan, K, (bt, sc, fmt), out, d_row, flags, rank_order=False)


def _stair_gemm(plan, K: int, packed, out: torch.Tensor, d_row: torch.Tensor, flags: int, *,
                rank_order: bool) -> None:
    """One staircase launch: rows scattered through the degree permutation into
    ``out`` (n rows), or with ``rank_order`` written in rank order to ``out``
    (rows0 rows) with ``d_row`` already in rank order."""
    bt, sc, fmt = packed
    dev = out.device
    lib = nat.load()
    st = _stream(dev)
    items, starts, n_cl, ws, fx = plan.schedule(K, dev)
    if plan.abits:
        flags |= nat.GC_HUB_A_BITS
    row_map = None if rank_order else plan.row_map.data_ptr()
    nat.check(_timed_call("hub_gemm", dev, lambda: lib.gc_hub_stair_gemm(
        plan._np_ptrs.ctypes.data, plan._np_rows.ctypes.data, plan._np_c0.ctypes.data,
        plan._np_w.ctypes.data, len(plan.steps), row_map, items.data_ptr(),
        starts.data_ptr(), n_cl, None if ws is None else ws.data_ptr(),
        None if fx is None else fx.data_ptr(), 0 if fx is None else fx.shape[0], bt.data_ptr(),
        plan.T, K, fmt, sc.data_ptr(), out.data_ptr(), _ld(out), d_row.data_ptr(), flags,
        st)), "hub_stair_gemm")


def tail_part(a: CsrMatrix, x: torch.Tensor, d: torch.Tensor, spec, out: torch.Tensor, *,
              d_row: torch.Tensor, values=None, relu=False, rows: tuple[int, int] | None = None,
              x_tail=None):
    """out (rows [lo, hi)) += the remaining edges (ReLU on the total).
    ``x_tail``: the gathered operand as fp16 rows (``sparse.HalfRows``, with
    the column scaling of the unit tail folded into its scales)."""
    plan = hub_plan(a, spec)
    lo, hi = rows if rows is not None else (0, a.n_rows)
    tail = plan.tail_block(values, lo, hi)
    if x_tail is not None:
        _spmm(tail, x_tail, weighted=values is not None,
              d_row=d_row[lo:hi] if values is None else None, relu=relu, out=out,
              accumulate=True, timer="spmm_tail")
    elif values is None:
        _spmm(tail, x, weighted=False, d_row=d_row[lo:hi], d_col=d, relu=relu, out=out,
              accumulate=True, timer="spmm_tail")
    else:
        _spmm(tail, x, weighted=True, relu=relu, out=out, accumulate=True, timer="spmm_tail")


def hybrid_aggregate(a: CsrMatrix, x: torch.Tensor, d: torch.Tensor, spec, *,
                     d_row: torch.Tensor | None = None, values: torch.Tensor | None = None,
                     relu: bool = False, out: torch.Tensor | None = None,
                     accumulate: bool = False, rows: tuple[int, int] | None = None,
                     packed: tuple | None = None, x_tail=None) -> torch.Tensor:
    """C = epi(D_row Ã D X) for a unit-valued pattern ``a`` via the dense/tail
    split ``spec`` (``d`` scales the columns — None when x already carries
    the column scaling; ``d_row`` the rows, default ``d`` itself for a square
    pattern).  ``values`` (optional) are a
    same-pattern matrix's values used for the tail instead of d_i·d_j (the
    precompute composition streams Ñ's values).  ``accumulate``: C += ...
    (ReLU on the total).  ``rows=(lo, hi)`` (block plans only) computes that
    row block (``out`` then has hi-lo rows); ``packed`` reuses one ``pack``;
    ``x_tail``: fp16 rows of x for the tail (see :func:`tail_part`)."""
    if isinstance(x, HalfRows):  # one fp16 operand for the dense part and the tail
        if x.shape[0] != a.n_cols:
            raise ShapeError("hybrid_aggregate: x must have n_cols rows")
        if d is not None and values is None:
            raise ShapeError("hybrid_aggregate: fp16 rows carry the column scaling (d=None)")
        x_tail = x
    elif x.dim() != 2 or x.shape[0] != a.n_cols or x.stride(1) != 1:
        raise ShapeError("hybrid_aggregate: x must be a row-major n_cols x K tensor")
    dev = _require_cuda(a.col_idx, x.xh if isinstance(x, HalfRows) else x)
    if d_row is None:
        if a.n_rows != a.n_cols or d is None:
            raise ShapeError("hybrid_aggregate: d_row is required for a rectangular pattern "
                             "or an already column-scaled x (d=None)")
        d_row = d
    K = x.shape[1]  # (HalfRows.shape is (n, K) too)
    lo, hi = rows if rows is not None else (0, a.n_rows)
    if out is None:
        if accumulate:
            raise ValueError("hybrid_aggregate: accumulate needs an output")
        out = torch.empty(hi - lo, K, dtype=torch.float32, device=dev)
    elif tuple(out.shape) != (hi - lo, K) or out.stride(1) != 1:
        raise ShapeError(f"hybrid_aggregate: out must be a row-major {hi - lo}x{K} tensor")

    def run():
        dense_part(a, x, d, spec, out, d_row=d_row, accumulate=accumulate, packed=packed,
                   rows=rows)
        tail_part(a, x, d, spec, out, d_row=d_row, values=values, relu=relu, rows=rows,
                  x_tail=x_tail)
        return 0

    _timed_call("spmm", dev, run)
    return out


def _candidates(K: int) -> list:
    """Staircase specs tried by the autotuner for this K.  (Block plans —
    ``HubPlan`` — never beat the staircase on the measured shapes; they stay
    reachable through GNNC_HUB_SPLIT=<T>.)"""
    if not nat.load().gc_hub_stair_supported(K):
        return []
    return [("stair", int(round(dl * 1000)), int(round(sl * 10))) for dl, sl in _stair_candidates(K)]


def _time_interleaved(runs: dict, rounds: int) -> dict:
    """Median CUDA-event time per run over ``rounds`` interleaved rounds, after
    one warm call each (clock / power-cap drift hits every candidate alike)."""
    for fn in runs.values():
        fn()
    samples: dict = {k: [] for k in runs}
    for _ in range(rounds):
        ev = {}
        for k, fn in runs.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            ev[k] = (e0, e1)
        torch.cuda.synchronize()
        for k, (e0, e1) in ev.items():
            samples[k].append(e0.elapsed_time(e1))
    return {k: float(sorted(v)[len(v) // 2]) for k, v in samples.items()}


def split_key(K: int, weighted: bool = False) -> tuple:
    """Cache key of the split choice: per K and operand term format of the
    current numerics class (a cell costs MMAs in proportion to the term
    count, so the classes choose separately).  Weighted (Ñ values, the
    precompute composition) and unit tails share the choice: the pattern and
    the dense part are the same, the tail differs by one value stream — one
    measurement per pattern keeps autotune noise from making the
    compositions differ by their splits rather than by their algebra."""
    del weighted
    return ("hubsplit-choice", int(K), term_format())


def choose_split(a: CsrMatrix, x: torch.Tensor, d: torch.Tensor, *,
                 d_row: torch.Tensor | None = None, values: torch.Tensor | None = None,
                 x_tail=None):
    """Split spec for (pattern, K): 0 (plain SpMM) unless a dense split is
    measurably faster, chosen on the first call and cached on the pattern.

    The candidates run as a tournament: each staircase plan is built (its
    block budget checked before allocation), timed against the current best
    in interleaved rounds, and the loser's blocks are freed at once — at most
    two plans are resident.  Device OOM while building or timing a candidate
    drops that candidate (the plain SpMM always remains).  Build time,
    autotune time and the peak extra device memory are recorded under
    ``a._plans[split_key(K, weighted) + ("stats",)]``."""
    import time

    mode = str(HUB_SPLIT)
    if mode == "0" or not a.has_unit_values:
        return 0
    if d_row is None:
        if a.n_rows != a.n_cols or d is None:
            return 0
        d_row = d
    if mode != "auto":
        spec = _parse_spec(mode)
        try:
            hub_plan(a, spec)
        except (ValueError, ShapeError):
            return 0  # the forced split does not fit this pattern
        return spec
    K = x.shape[1]
    key = split_key(K, values is not None)
    if key in a._plans:
        return a._plans[key]
    if isinstance(x, HalfRows):
        x_tail = x
    elif x.stride(1) != 1:
        a._plans[key] = 0
        return 0
    if a.nnz < HUB_MIN_NNZ:
        a._plans[key] = 0
        return 0
    cands = _candidates(K)
    if not cands:
        a._plans[key] = 0
        return 0
    dev = x.device
    t_start = time.perf_counter()
    torch.cuda.synchronize(dev)
    mem0 = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    scratch = torch.empty(a.n_rows, K, dtype=torch.float32, device=dev)
    src = a if values is None else a.with_values(values)

    def plain():
        if x_tail is not None:
            _spmm(src, x_tail, weighted=values is not None,
                  d_row=None if values is not None else d_row, out=scratch, timer=None)
            return
        _spmm(src, x, weighted=values is not None, d_row=None if values is not None else d_row,
              d_col=None if values is not None else d, out=scratch, timer=None)

    def hybrid(spec):
        return lambda: hybrid_aggregate(a, x, d, spec, d_row=d_row, values=values, out=scratch,
                                        x_tail=x_tail)

    best, times, build_s = 0, {}, 0.0
    for spec in cands:
        try:
            t0 = time.perf_counter()
            hub_plan(a, spec)
            torch.cuda.synchronize(dev)
            build_s += time.perf_counter() - t0
            runs = {best: plain if best == 0 else hybrid(best), spec: hybrid(spec)}
            tt = _time_interleaved(runs, AUTOTUNE_ROUNDS)
        except ValueError:
            continue  # no step pays for its cells, or over the block budget
        except torch.cuda.OutOfMemoryError:
            a._plans.pop(("hubsplit", spec), None)
            torch.cuda.empty_cache()
            continue
        times.update(tt)
        # a split must be clearly (> 3 %) faster than the plain SpMM
        win = tt[spec] < tt[best] and (best != 0 or tt[spec] < 0.97 * tt[0])
        loser = best if win else spec
        if win:
            best = spec
        if loser != 0:
            a._plans.pop(("hubsplit", loser), None)  # free its blocks now
    del scratch
    torch.cuda.synchronize(dev)
    a._plans[key] = best
    a._plans[key + ("times",)] = {spec_label(s): round(t, 4) for s, t in times.items()}
    a._plans[key + ("stats",)] = {
        "plan_build_s": round(build_s, 3),
        "autotune_s": round(time.perf_counter() - t_start, 3),
        "peak_extra_bytes": int(torch.cuda.max_memory_allocated(dev) - mem0),
        "resident_plan_bytes": int(hub_plan(a, best).cells * (0.125 if HUB_ABITS else 2)) if best else 0}
    return best
