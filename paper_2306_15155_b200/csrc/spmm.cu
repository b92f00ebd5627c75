// CSR SpMM for sm_100a: C = epi( D_row * (A ∘ d_col) * B ), and its GAT form
// C = epi( softmax_row(LeakyReLU(s_i + t_j)) * B ) with the edge softmax
// computed online inside the aggregation (α is never written).
//
// Reference semantics: gnncompose/sparse.py:196-219 (_spmm_kernel,
// _spmm_unweighted_kernel) and gat.py:72-95 + sparse.py:196-205 for the GAT
// form.  A row is owned by a group of LPR lanes; each lane owns NV float4 (or
// scalar) column slots of the row and accumulates the row's edges in storage
// order with FMA, so the order is fixed and `values == nullptr` is
// bit-identical to unit values.
//
// Memory plan: col_idx/values stream once (evict-first),
// the gathered rows of B go through the read-only path as 128-bit loads, the
// next batch of column indices is in flight while the current batch's rows are
// gathered, and U edges are unrolled per step.  The D^-1/2 factors of the
// dynamic composition are folded in (d_col into the edge weight, d_row into
// the epilogue) instead of materialising D^-1/2 H.  Heavy rows are cut into
// plan items whose partial sums (and, for GAT, partial (max, sum) pairs) are
// merged in slot order by the fixup kernel.
#include <algorithm>

#include <cuda_fp16.h>

#include "common.cuh"

namespace gnnc {
namespace {

constexpr int kThreads = 256;
// resident CTAs per SM the SpMM kernel is compiled for (register cap
// 65536 / (kThreads * GNNC_SPMM_MINB)); the gathers are latency-bound, so
// warps in flight matter
#ifndef GNNC_SPMM_MINB
#define GNNC_SPMM_MINB 1
#endif
// the same for the fp16-row (GC_SPMM_B_F16) instances (SDDMM-score GAT
// rows hold the score operands too: half as many), and their edges unrolled
// per step (16-byte chunks in flight per lane = U x NV/2).  Measured on
// Reddit / products K = 256 (profiles/data/ab_bh_unroll_r02.json): U = 4 at
// 4 CTAs/SM 1.65 / 7.68 ms per layer, U = 8 at 1 CTA/SM (96 registers)
// 1.99 / 8.79 ms — the gathers need warps in flight more than chunks per lane.
#ifndef GNNC_SPMM_BH_MINB
#define GNNC_SPMM_BH_MINB 4
#endif
// one 16-byte chunk per lane, one row per warp (LPR = 32, NV = 2, the
// unpredicated loop): 40 registers, 6 CTAs/SM — the gathers
// are latency-bound (long-scoreboard stalls), so warps in flight pay:
// Reddit tail 0.96 -> 0.84 ms, products 6.9 -> 6.0 ms per layer over 4 CTAs
// (profiles/data/ab_occupancy_r02.json)
#ifndef GNNC_SPMM_BH_MINB1
#define GNNC_SPMM_BH_MINB1 6
#endif
// (the GAT reassoc aggregation runs 5 CTAs/SM at 47 registers: its
// online-softmax state spills at 40 — arxiv K = 256 0.47 ms at 6 CTAs,
// 0.33 at 4, 0.31 at 5; products 8.26 -> 7.72 ms from 4 to 5)
#ifndef GNNC_SPMM_BH_MINB1_GAT
#define GNNC_SPMM_BH_MINB1_GAT 5
#endif
// fp16-weight FMA (fma.rn.f32.f16) for batches whose weights are exact in
// fp16; 0 keeps widen + FFMA everywhere (A/B builds)
#ifndef GNNC_SPMM_F16W
#define GNNC_SPMM_F16W 1
#endif
#ifndef GNNC_SPMM_BH_U
#define GNNC_SPMM_BH_U 4
#endif

struct SpmmArgs {
  const int32_t *row_ptr;
  const int32_t *col_idx;
  const float *values;
  const float *d_row;
  const float *d_col;
  const float *B;
  int64_t ldb;
  int64_t K;
  float *C;
  int64_t ldc;
  const int4 *items;  // nullptr: one item per row
  int64_t n_items;
  float *partial;     // [n_slots][K] for split items
  float2 *partial_mz; // GAT: [n_slots] running (max, sum) of each split item
  const float *s;     // GAT: per-row source score (s = HW a_src)
  const float *t;     // GAT: per-column target score (t = HW a_dst)
  float slope;        // GAT: LeakyReLU slope
  const float *a_src; // GAT-SDDMM: attention vectors (length K): e = a_src.B_i + a_dst.B_j
  const float *a_dst;
  uint32_t flags;
  bool hints;         // col_idx carries hub tags in bit 31 (gc_tag_hub_columns)
  const float *B_self; // GAT-SDDMM: row i's own features (a_src.B_self[i]); B for a square
  int64_t ld_self;     //   pattern, a rank's own rows for a row block of a partition
  int sig_ld;          // fp16 rows: scales per row (> 1: one per 256-column pass, d_col is
                       //   n_cols x sig_ld and pass blockIdx.y reads column blockIdx.y)
};

template <bool VEC>
struct Lanes;
template <>
struct Lanes<true> {
  using T = float4;
  static constexpr int W = 4;
};
template <>
struct Lanes<false> {
  using T = float;
  static constexpr int W = 1;
};

__device__ __forceinline__ float4 zero_of(float4) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float zero_of(float) { return 0.f; }
__device__ __forceinline__ void fma_into(float4 &acc, float w, float4 b) {
  // (packed FFMA2 measured no faster: the operand packing costs the issue
  // slots it saves — profiles/data/ab_ffma2_r02.json)
  acc.x = fmaf(w, b.x, acc.x);
  acc.y = fmaf(w, b.y, acc.y);
  acc.z = fmaf(w, b.z, acc.z);
  acc.w = fmaf(w, b.w, acc.w);
}
__device__ __forceinline__ void fma_into(float &acc, float w, float b) { acc = fmaf(w, b, acc); }
__device__ __forceinline__ float dot_of(float4 x, float4 w) {
  return fmaf(x.x, w.x, fmaf(x.y, w.y, fmaf(x.z, w.z, x.w * w.w)));
}
__device__ __forceinline__ float dot_of(float x, float w) { return x * w; }
__device__ __forceinline__ void scale_into(float4 &acc, float sc) {
  acc.x *= sc, acc.y *= sc, acc.z *= sc, acc.w *= sc;
}
__device__ __forceinline__ void scale_into(float &acc, float sc) { acc *= sc; }
__device__ __forceinline__ void load_b(float4 &dst, const float *p) { dst = ldg_f4(p); }
__device__ __forceinline__ void load_b(float &dst, const float *p) { dst = __ldg(p); }
// hot-column hint (bit 31 of a tagged col_idx entry): hub rows are kept in L1
__device__ __forceinline__ void load_b_hint(float4 &dst, const float *p, bool hot) {
  dst = hot ? ldg_f4_keep(p) : ldg_f4_stream(p);
}
__device__ __forceinline__ void load_b_hint(float &dst, const float *p, bool) { dst = __ldg(p); }
// fp16 operand rows (GC_SPMM_B_F16): one 16-byte load = eight halves = two
// adjacent float4 column slots, widened to fp32 in registers (exact)
__device__ __forceinline__ uint4 ldg_u4(const char *p) {
  uint4 r;
  asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
__device__ __forceinline__ float2 h2f(uint32_t q) {
  return __half22float2(*reinterpret_cast<const __half2 *>(&q));
}
__device__ __forceinline__ void widen_h8(uint4 q, float4 &lo4, float4 &hi4) {
  const float2 a = h2f(q.x), b = h2f(q.y), c = h2f(q.z), d = h2f(q.w);
  lo4 = make_float4(a.x, a.y, b.x, b.y);
  hi4 = make_float4(c.x, c.y, d.x, d.y);
}

// a0 += w * q.lo, a1 += w * q.hi with w and q's halves fp16, a0/a1 fp32
// (sm_100 mixed-precision FMA: the fp16 product is exact, one rounding)
__device__ __forceinline__ void fma_h2(float &a0, float &a1, uint32_t w, uint32_t q) {
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %3;\n\t"
      "fma.rn.f32.f16 %0, %2, l, %0;\n\tfma.rn.f32.f16 %1, %2, h, %1;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "h"((unsigned short)w), "r"(q));
}

__device__ __forceinline__ float epi1(float v, float ds, float old, uint32_t flags) {
  v *= ds;
  if (flags & GC_ACCUMULATE) v += old;
  if (flags & GC_RELU) v = fmaxf(v, 0.0f);
  return v;
}

// Column of lane gl's slot v.  BH (fp16 rows): slots 2u and 2u+1 are the two
// halves of one 8-column (16-byte) chunk, so each gather is a full 16-byte
// load; otherwise slot v holds 4 columns at stride 4·LPR.
template <int LPR, int NV, bool VEC, bool BH = false>
__device__ __forceinline__ int64_t col_of(int64_t c0, int v, int gl) {
  if (BH) return c0 + (int64_t)(v >> 1) * LPR * 8 + gl * 8 + (v & 1) * 4;
  return VEC ? c0 + (int64_t)v * LPR * 4 + gl * 4 : c0 + (int64_t)v * LPR + gl;
}

template <int LPR, int NV, bool VEC, bool BH = false>
__device__ __forceinline__ void store_row(const SpmmArgs &a, int row, int slot, int gl,
                                          int64_t c0, float ds,
                                          const typename Lanes<VEC>::T (&acc)[NV]) {
  const uint32_t flags = a.flags;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int64_t c = col_of<LPR, NV, VEC, BH>(c0, v, gl);
    if (c >= a.K) continue;
    if (slot >= 0) {  // raw partial sum, combined later by spmm_fixup
      float *dst = a.partial + (int64_t)slot * a.K + c;
      if constexpr (VEC) stg_f4(dst, acc[v]);
      else *dst = acc[v];
      continue;
    }
    float *dst = a.C + (int64_t)row * a.ldc + c;
    if constexpr (VEC) {
      float4 old = make_float4(0.f, 0.f, 0.f, 0.f);
      if (flags & GC_ACCUMULATE) old = *reinterpret_cast<const float4 *>(dst);
      float4 r;
      r.x = epi1(acc[v].x, ds, old.x, flags);
      r.y = epi1(acc[v].y, ds, old.y, flags);
      r.z = epi1(acc[v].z, ds, old.z, flags);
      r.w = epi1(acc[v].w, ds, old.w, flags);
      stg_f4(dst, r);
    } else {
      const float old = (flags & GC_ACCUMULATE) ? *dst : 0.f;
      *dst = epi1(acc[v], ds, old, flags);
    }
  }
}

// One group of LPR lanes per work item (a row, or a chunk of a heavy row).
// MODE 0: SpMM.  MODE 1: GAT, e = LeakyReLU(s_i + t_j) with t_j gathered.
// MODE 2: GAT whose score is an SDDMM over the gathered rows themselves,
// e = LeakyReLU(a_src.B_i + a_dst.B_j): one gather of B_j feeds both the
// score and the aggregation (needs the whole row in one column pass).
// BH (MODE 0 only): B holds fp16 rows (GC_SPMM_B_F16, the TF32 class's
// half-width gather operand), half the gathered bytes per edge.
template <int LPR, int NV, bool VEC, bool HAS_VAL, bool HAS_DCOL, int MODE, bool HINT,
          bool BH = false>
// (fp32 rows with <= 2 slots: 4 CTAs/SM for the SpMM, 3 for the GAT modes —
// the round-1 build's occupancy; at their natural 80-100 registers they ran
// one CTA/SM fewer, the SDDMM-score mode 35 % slower on arxiv; wider rows
// keep their registers, capping them spills)
__global__ void __launch_bounds__(kThreads, BH ? (MODE == 2 ? (GNNC_SPMM_BH_MINB + 1) / 2
                                                         : LPR == 32 && NV == 2
                                                               ? (MODE == 0 ? GNNC_SPMM_BH_MINB1
                                                                            : GNNC_SPMM_BH_MINB1_GAT)
                                                               : GNNC_SPMM_BH_MINB)
                                              : (NV > 2 ? GNNC_SPMM_MINB : MODE == 0 ? 4 : 3))
    spmm_kernel(const SpmmArgs a) {
  static_assert(!BH || (!HINT && VEC && NV % 2 == 0),
                "fp16 operand rows: no L1 tags, 16-byte chunks of two slots");
  // GAT modes with fp16 rows: the row scale sigma_j (a.d_col) is gathered
  // per edge beside t_j; it scales the gathered row in the score (SD) and
  // in the aggregation, never the softmax denominator
  constexpr bool SIG = BH && MODE != 0;
  using T = typename Lanes<VEC>::T;
  constexpr bool GAT = MODE != 0;
  constexpr bool SD = MODE == 2;
  constexpr int GPB = kThreads / LPR;
  // edges unrolled per step: ~8 independent 16-byte gathers in flight per lane
  // (never more than LPR: the edge batch is shuffled within the lane group)
  // (BH: one 16-byte load covers two slots, so count loads, not slots)
  constexpr int NVL = BH ? NV / 2 : NV;
  constexpr int U0 = BH ? (GNNC_SPMM_BH_U / NVL > 0 ? GNNC_SPMM_BH_U / NVL : 1)
                        : NVL >= 8 ? 1 : NVL >= 4 ? 2 : NVL >= 2 ? 4 : 8;
  constexpr int U = U0 < LPR ? U0 : LPR;
  static_assert(LPR % U == 0, "an edge batch of LPR lanes is consumed U edges at a time");
  const int g = threadIdx.x / LPR;
  const int gl = threadIdx.x % LPR;
  const int64_t item = (int64_t)blockIdx.x * GPB + g;
  const bool live = item < a.n_items;

  int row = 0, beg = 0, end = 0, slot = -1;
  if (live) {
    if (a.items) {
      const int4 it = __ldg(a.items + item);
      row = it.x, beg = it.y, end = it.z, slot = it.w;
    } else {
      row = (int)item;
      beg = __ldg(a.row_ptr + row);
      end = __ldg(a.row_ptr + row + 1);
    }
  }
  constexpr int64_t kColsPerPass = (int64_t)LPR * NV * Lanes<VEC>::W;
  const int64_t c0 = (int64_t)blockIdx.y * kColsPerPass;
  // d_col index of column j: per row, or per (row, 256-column pass) for fp16
  // rows with chunked scales (the entry points check kColsPerPass == 256)
  const int64_t sig_ld = a.sig_ld > 1 ? a.sig_ld : 1;
  const int64_t sig_off = a.sig_ld > 1 ? (int64_t)blockIdx.y : 0;
  auto sig_at = [&](int j) -> int64_t { return (int64_t)j * sig_ld + sig_off; };

  // column slots of this lane (32-bit: K is a feature width, far below 2^31)
  bool colok[NV];
  int coff[NV];
  const int kcols = (int)a.K;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    coff[v] = (int)col_of<LPR, NV, VEC, BH>(c0, v, gl);
    colok[v] = coff[v] < kcols;
  }

  T acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = zero_of(T{});
  constexpr int kSlotStride = LPR * Lanes<VEC>::W;  // floats between a lane's column slots
  constexpr int ESZ = BH ? 2 : 4;  // bytes per operand element
  // FLAT (fp16 rows, one group per warp, one 16-byte chunk per lane): lanes
  // whose columns lie past K gather column 0 instead (never stored), so the
  // inner loop carries no column predicate
  constexpr bool FLATC = BH && MODE != 2 && LPR == 32 && NV == 2;
  const int cbase = (FLATC && !colok[0]) ? 0 : coff[0];
  const char *bbase = reinterpret_cast<const char *>(a.B) + (int64_t)cbase * ESZ;
  const uint32_t ldb_bytes = (uint32_t)(a.ldb * ESZ);

  const int len = end - beg;
  const int wmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)len);
  // GAT: online softmax state; m is identical on every lane of the group,
  // zl sums this lane's own edge weights relative to m.
  float si = (MODE == 1 && live) ? __ldg(a.s + row) : 0.0f;
  float gs1 = 1.0f;  // SIG: sigma of this lane's edge in the next batch
  float m = -INFINITY, zl = 0.0f;
  T adst[NV];
  if constexpr (SD) {  // source term a_src.B_i and this lane's slice of a_dst
    float part = 0.0f;
    const float *bi = a.B_self + (int64_t)row * a.ld_self;
#pragma unroll
    for (int vv = 0; vv < NV; ++vv) {
      adst[vv] = zero_of(T{});
      if (colok[vv]) {
        T x, w;
        load_b(w, a.a_src + coff[vv]);
        if (live) {
          load_b(x, bi + coff[vv]);
          part += dot_of(x, w);
        }
        load_b(adst[vv], a.a_dst + coff[vv]);
      }
    }
    si = group_sum<LPR>(part);
  }
  // Two-deep software pipeline over batches of LPR edges: while batch i's rows
  // of B are gathered, batch i+1's per-node gather (d_j or t_j) and batch
  // i+2's (col, value) loads are already in flight.
  constexpr bool NEEDG = HAS_DCOL || MODE == 1;
  int j1 = 0, j2 = 0;
  float v1 = 1.0f, v2 = 1.0f, g1 = 0.0f;
  if (gl < len) {
    j1 = ldg_stream_i32(a.col_idx + beg + gl);
    if (HAS_VAL) v1 = ldg_stream_f32(a.values + beg + gl);
    if (NEEDG)
      g1 = __ldg(MODE == 1 ? a.t + (HINT ? (j1 & 0x7FFFFFFF) : j1)
                           : a.d_col + sig_at(HINT ? (j1 & 0x7FFFFFFF) : j1));
    if (SIG) gs1 = __ldg(a.d_col + sig_at(j1));
  }
  if (LPR + gl < len) {
    j2 = ldg_stream_i32(a.col_idx + beg + LPR + gl);
    if (HAS_VAL) v2 = ldg_stream_f32(a.values + beg + LPR + gl);
  }
  // fp16 rows, one row per warp: the edge loop runs unpredicated
  // (fp32 rows measured ~1 % slower unpredicated — the fp32 class at Reddit
  // K = 256, 2.70 vs 2.68 ms — so they keep the predicated loop)
  constexpr bool FLAT = BH && MODE != 2 && LPR == 32;
  if constexpr (FLAT) {
    // unpredicated gathers (FLAT below): lanes past the row's end gather
    // one of the row's own columns, so no other row's values enter it
    const int j0 = __shfl_sync(0xffffffffu, j1, 0);
    if (gl >= len) j1 = j0;
    if (LPR + gl >= len) j2 = j0;
  }
  for (int base = 0; base < wmax; base += LPR) {
    const int j = HINT ? (j1 & 0x7FFFFFFF) : j1;  // HINT: bit 31 tags a hub column
    const bool hot = HINT && j1 < 0;
    const float v = v1;
    const float g = g1;
    const float gsig = gs1;
    const bool mine = base + gl < len;
    j1 = j2;
    v1 = v2;
    if (NEEDG && base + LPR + gl < len)
      g1 = __ldg(MODE == 1 ? a.t + (HINT ? (j1 & 0x7FFFFFFF) : j1)
                           : a.d_col + sig_at(HINT ? (j1 & 0x7FFFFFFF) : j1));
    if (SIG && base + LPR + gl < len) gs1 = __ldg(a.d_col + sig_at(j1));
    if (base + 2 * LPR + gl < len) {
      j2 = ldg_stream_i32(a.col_idx + beg + base + 2 * LPR + gl);
      if (HAS_VAL) v2 = ldg_stream_f32(a.values + beg + base + 2 * LPR + gl);
    }
    float dj = 1.0f;
    if (HAS_DCOL && mine) dj = g;
    float e = -INFINITY;
    if (MODE == 1) {
      if (mine) e = leaky(si + g, a.slope);
      const float mb = group_max<LPR>(e);
      const float mn = fmaxf(m, mb);
      if (mn > m) {  // group-uniform: rescale the running sums to the new max
        const float sc = __expf(m - mn);
#pragma unroll
        for (int vv = 0; vv < NV; ++vv) scale_into(acc[vv], sc);
        zl *= sc;
        m = mn;
      }
      dj = mine ? __expf(e - m) : 0.0f;
      zl += dj;
    }
    // fp16 weights (MODE 0, fp16 rows): when every weight of the batch is
    // exact in fp16 — unit values times a power-of-two row scale sigma_j —
    // the FMA takes the fp16 element directly (fma.rn.f32.f16: a product of
    // two fp16 values is exact in fp32, so the sum is bit-identical to the
    // widen + FFMA path, one instruction per element instead of two)
    bool hw = false;
    uint32_t wh = 0;
    if constexpr (BH && MODE == 0 && GNNC_SPMM_F16W) {
      const float w = mine ? v * dj : 0.0f;
      const __half h = __float2half_rn(w);
      wh = __half_as_ushort(h);
      hw = __all_sync(0xffffffffu, __half2float(h) == w);
    }
    const int cnt = len - base;  // edges left for this group (may be <= 0)
    const int cntw = min(LPR, wmax - base);
#pragma unroll 1
    for (int e0 = 0; e0 < cntw; e0 += U) {
      if constexpr (BH) {
        // fp16 rows: U edges x NV/2 raw 16-byte chunks in flight (4
        // registers each); each chunk is widened to fp32 where it is used
        // (never all at once: that would double the live registers)
        constexpr int NVH = NV / 2;
        // one group per warp (SpMM and GAT reassoc): past the row's end a
        // lane gathers one of the row's own columns with weight 0, so the
        // gathers and FMAs run unpredicated (adding 0 leaves acc unchanged)
        uint4 rw[U][NVH];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int je = __shfl_sync(0xffffffffu, j, e0 + u, LPR);
          const bool ok = FLAT || (e0 + u) < cnt;
          const char *brow_c = bbase + (uint64_t)(uint32_t)je * ldb_bytes;
#pragma unroll
          for (int c = 0; c < NVH; ++c)
            if (ok && (FLATC || colok[2 * c]))
              rw[u][c] = ldg_u4(brow_c + (coff[2 * c] - coff[0]) * ESZ);
        }
        if constexpr (SD) {
          float eu[U], su[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            su[u] = SIG ? __shfl_sync(0xffffffffu, gsig, e0 + u, LPR) : 1.0f;
            float part = 0.0f;
#pragma unroll
            for (int c = 0; c < NVH; ++c) {
              if ((e0 + u) < cnt && colok[2 * c]) {
                float4 lo4, hi4;
                widen_h8(rw[u][c], lo4, hi4);
                part += dot_of(lo4, adst[2 * c]) + dot_of(hi4, adst[2 * c + 1]);
              }
            }
            part = group_sum<LPR>(part) * su[u];
            eu[u] = (e0 + u) < cnt ? leaky(si + part, a.slope) : -INFINITY;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if ((e0 + u) < cnt) {
              if (eu[u] > m) {
                const float sc = __expf(m - eu[u]);
#pragma unroll
                for (int vv = 0; vv < NV; ++vv) scale_into(acc[vv], sc);
                zl *= sc;
                m = eu[u];
              }
              const float w = __expf(eu[u] - m);
              zl += w;
              const float wa = w * su[u];
#pragma unroll
              for (int c = 0; c < NVH; ++c) {
                if (colok[2 * c]) {
                  float4 lo4, hi4;
                  widen_h8(rw[u][c], lo4, hi4);
                  fma_into(acc[2 * c], wa, lo4);
                  fma_into(acc[2 * c + 1], wa, hi4);
                }
              }
            }
          }
        } else if (MODE == 0 && hw) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t we = __shfl_sync(0xffffffffu, wh, e0 + u, LPR);
            if (FLAT || (e0 + u) < cnt) {
#pragma unroll
              for (int c = 0; c < NVH; ++c) {
                if (FLATC || colok[2 * c]) {
                  fma_h2(acc[2 * c].x, acc[2 * c].y, we, rw[u][c].x);
                  fma_h2(acc[2 * c].z, acc[2 * c].w, we, rw[u][c].y);
                  fma_h2(acc[2 * c + 1].x, acc[2 * c + 1].y, we, rw[u][c].z);
                  fma_h2(acc[2 * c + 1].z, acc[2 * c + 1].w, we, rw[u][c].w);
                }
              }
            }
          }
        } else {
          const float w = mine ? v * dj * (SIG ? gsig : 1.0f) : 0.0f;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const float we = __shfl_sync(0xffffffffu, w, e0 + u, LPR);
            if (FLAT || (e0 + u) < cnt) {
#pragma unroll
              for (int c = 0; c < NVH; ++c) {
                if (FLATC || colok[2 * c]) {
                  float4 lo4, hi4;
                  widen_h8(rw[u][c], lo4, hi4);
                  fma_into(acc[2 * c], we, lo4);
                  fma_into(acc[2 * c + 1], we, hi4);
                }
              }
            }
          }
        }
        continue;
      }
      T bv[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int je = __shfl_sync(0xffffffffu, j, e0 + u, LPR);
        const bool ok = FLAT || (e0 + u) < cnt;
        const float *brow = reinterpret_cast<const float *>(
            bbase + (uint64_t)(uint32_t)je * ldb_bytes);
        bool hote = false;
        if (HINT) hote = __shfl_sync(0xffffffffu, (int)hot, e0 + u, LPR) != 0;
#pragma unroll
        for (int vv = 0; vv < NV; ++vv) {
          if (ok && colok[vv]) {
            if (HINT) load_b_hint(bv[u][vv], brow + vv * kSlotStride, hote);
            else load_b(bv[u][vv], brow + vv * kSlotStride);
          }
        }
      }
      if constexpr (SD) {
        // per-edge score from the row just gathered, then an online-softmax
        // update in edge order (m, zl identical on every lane of the group)
        float eu[U], su[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          su[u] = SIG ? __shfl_sync(0xffffffffu, gsig, e0 + u, LPR) : 1.0f;
          float part = 0.0f;
#pragma unroll
          for (int vv = 0; vv < NV; ++vv)
            if ((e0 + u) < cnt && colok[vv]) part += dot_of(bv[u][vv], adst[vv]);
          part = group_sum<LPR>(part) * su[u];
          eu[u] = (e0 + u) < cnt ? leaky(si + part, a.slope) : -INFINITY;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if ((e0 + u) < cnt) {
            if (eu[u] > m) {
              const float sc = __expf(m - eu[u]);
#pragma unroll
              for (int vv = 0; vv < NV; ++vv) scale_into(acc[vv], sc);
              zl *= sc;
              m = eu[u];
            }
            const float w = __expf(eu[u] - m);
            zl += w;
            const float wa = w * su[u];
#pragma unroll
            for (int vv = 0; vv < NV; ++vv)
              if (colok[vv]) fma_into(acc[vv], wa, bv[u][vv]);
          }
        }
      } else {
        // unit weights (value-blind, no d_j): no weight shuffle; fma(1, b, acc)
        // rounds exactly like the weighted kernel with unit values
        constexpr bool UNIT = !HAS_VAL && !HAS_DCOL && MODE == 0;
        const float w = mine ? v * dj * (SIG ? gsig : 1.0f) : 0.0f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float we = UNIT ? 1.0f : __shfl_sync(0xffffffffu, w, e0 + u, LPR);
          if (FLAT || (e0 + u) < cnt) {
#pragma unroll
            for (int vv = 0; vv < NV; ++vv)
              if (colok[vv]) fma_into(acc[vv], we, bv[u][vv]);
          }
        }
      }
    }
  }
  float ds = 1.0f;
  if (GAT) {
    const float z = SD ? zl : group_sum<LPR>(zl);  // SD: every lane already holds the row sum
    if (slot >= 0) {
      if (live && gl == 0 && blockIdx.y == 0) a.partial_mz[slot] = make_float2(m, z);
    } else {
      ds = z > 0.0f ? 1.0f / z : 0.0f;  // rows without edges aggregate to 0
    }
  } else if (slot < 0 && live && a.d_row) {
    ds = __ldg(a.d_row + row);
  }
  if (live) store_row<LPR, NV, VEC, BH>(a, row, slot, gl, c0, ds, acc);
}

// Combine the partial sums of split rows in slot order, then the epilogue.
template <int LPR, int NV, bool VEC, int MODE>
__global__ void __launch_bounds__(kThreads)
    spmm_fixup_kernel(const SpmmArgs a, const int4 *split_rows, int64_t n_split) {
  using T = typename Lanes<VEC>::T;
  constexpr bool GAT = MODE != 0;
  constexpr int GPB = kThreads / LPR;
  const int g = threadIdx.x / LPR;
  const int gl = threadIdx.x % LPR;
  const int64_t r = (int64_t)blockIdx.x * GPB + g;
  if (r >= n_split) return;
  const int4 sr = __ldg(split_rows + r);
  constexpr int64_t kColsPerPass = (int64_t)LPR * NV * Lanes<VEC>::W;
  const int64_t c0 = (int64_t)blockIdx.y * kColsPerPass;
  T acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = zero_of(T{});
  float mx = -INFINITY, z = 0.0f;
  if (GAT)
    for (int q = 0; q < sr.z; ++q) mx = fmaxf(mx, a.partial_mz[sr.y + q].x);
  for (int q = 0; q < sr.z; ++q) {
    const float *src = a.partial + (int64_t)(sr.y + q) * a.K;
    float w = 1.0f;
    if (GAT) {
      const float2 mz = a.partial_mz[sr.y + q];
      w = mz.x == -INFINITY ? 0.0f : __expf(mz.x - mx);
      z = fmaf(w, mz.y, z);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int64_t c = col_of<LPR, NV, VEC>(c0, v, gl);
      if (c < a.K) {
        T t;
        load_b(t, src + c);
        fma_into(acc[v], w, t);
      }
    }
  }
  float ds = 1.0f;
  if (GAT) ds = z > 0.0f ? 1.0f / z : 0.0f;
  else if (a.d_row) ds = __ldg(a.d_row + sr.x);
  store_row<LPR, NV, VEC>(a, sr.x, -1, gl, c0, ds, acc);
}

template <int LPR, int NV, bool VEC, int MODE, bool BH = false>
int launch_cfg(const SpmmArgs &a, const int4 *split_rows, int64_t n_split, cudaStream_t st) {
  constexpr int GPB = kThreads / LPR;
  constexpr int64_t kColsPerPass = (int64_t)LPR * NV * Lanes<VEC>::W;
  const int64_t ychunks = (a.K + kColsPerPass - 1) / kColsPerPass;
  if (ychunks > 65535) {
    set_error("gc_spmm_f32: K=%lld too large", (long long)a.K);
    return GC_ERR_UNSUPPORTED;
  }
  if (a.n_items > 0) {
    dim3 grid((unsigned)((a.n_items + GPB - 1) / GPB), (unsigned)ychunks);
    const bool hv = a.values != nullptr, hd = a.d_col != nullptr;
    if constexpr (BH && MODE != 0) {
      spmm_kernel<LPR, NV, VEC, false, false, MODE, false, true><<<grid, kThreads, 0, st>>>(a);
    } else if constexpr (BH) {
      if (hv && hd) spmm_kernel<LPR, NV, VEC, true, true, 0, false, true><<<grid, kThreads, 0, st>>>(a);
      else if (hv) spmm_kernel<LPR, NV, VEC, true, false, 0, false, true><<<grid, kThreads, 0, st>>>(a);
      else if (hd) spmm_kernel<LPR, NV, VEC, false, true, 0, false, true><<<grid, kThreads, 0, st>>>(a);
      else spmm_kernel<LPR, NV, VEC, false, false, 0, false, true><<<grid, kThreads, 0, st>>>(a);
    } else if constexpr (MODE != 0) {
      if (a.hints) spmm_kernel<LPR, NV, VEC, false, false, MODE, true><<<grid, kThreads, 0, st>>>(a);
      else spmm_kernel<LPR, NV, VEC, false, false, MODE, false><<<grid, kThreads, 0, st>>>(a);
    } else if (a.hints) {
      if (hv && hd) spmm_kernel<LPR, NV, VEC, true, true, 0, true><<<grid, kThreads, 0, st>>>(a);
      else if (hv) spmm_kernel<LPR, NV, VEC, true, false, 0, true><<<grid, kThreads, 0, st>>>(a);
      else if (hd) spmm_kernel<LPR, NV, VEC, false, true, 0, true><<<grid, kThreads, 0, st>>>(a);
      else spmm_kernel<LPR, NV, VEC, false, false, 0, true><<<grid, kThreads, 0, st>>>(a);
    } else {
      if (hv && hd) spmm_kernel<LPR, NV, VEC, true, true, 0, false><<<grid, kThreads, 0, st>>>(a);
      else if (hv) spmm_kernel<LPR, NV, VEC, true, false, 0, false><<<grid, kThreads, 0, st>>>(a);
      else if (hd) spmm_kernel<LPR, NV, VEC, false, true, 0, false><<<grid, kThreads, 0, st>>>(a);
      else spmm_kernel<LPR, NV, VEC, false, false, 0, false><<<grid, kThreads, 0, st>>>(a);
    }
    int rc = check_launch(MODE == 0   ? "spmm_kernel"
                          : MODE == 1 ? "gat_aggregate_kernel"
                                      : "gat_sddmm_aggregate_kernel");
    if (rc) return rc;
  }
  if (n_split > 0) {
    dim3 grid((unsigned)((n_split + GPB - 1) / GPB), (unsigned)ychunks);
    spmm_fixup_kernel<LPR, NV, VEC, MODE><<<grid, kThreads, 0, st>>>(a, split_rows, n_split);
    return check_launch("spmm_fixup_kernel");
  }
  return GC_OK;
}

}  // namespace

namespace {

template <int MODE>
int dispatch(SpmmArgs &a, int64_t n_rows, int algo, const int32_t *items, int64_t n_items,
             const int32_t *split_rows, int64_t n_split_rows, void *workspace, size_t ws_bytes,
             void *stream, const char *who) {
  const int4 *sr = nullptr;
  int64_t n_split = 0;
  if (algo == GC_SPMM_NNZ_SPLIT) {
    GC_REQUIRE(items && n_items >= n_rows, GC_ERR_VALUE, "%s: NNZ_SPLIT needs a plan", who);
    GC_REQUIRE(n_split_rows == 0 || split_rows, GC_ERR_VALUE, "%s: split_rows null", who);
    a.items = reinterpret_cast<const int4 *>(items);
    a.n_items = n_items;
    sr = reinterpret_cast<const int4 *>(split_rows);
    n_split = n_split_rows;
    if (n_split > 0) {
      GC_REQUIRE(workspace != nullptr && aligned16(workspace), GC_ERR_WORKSPACE,
                 "%s: 16-byte aligned workspace required", who);
      a.partial = static_cast<float *>(workspace);
      if (MODE != 0) {
        // (max, sum) pairs follow the [n_slots][K] partial rows; the host
        // wrapper sized the workspace from the plan it owns.
        GC_REQUIRE(ws_bytes > 0, GC_ERR_WORKSPACE, "%s: bad workspace", who);
        const size_t n_slots = ws_bytes / (size_t)(4 * a.K + 8);
        const size_t off = (n_slots * (size_t)a.K * 4 + 7) & ~(size_t)7;
        a.partial_mz = reinterpret_cast<float2 *>(static_cast<char *>(workspace) + off);
      }
    }
  } else if (algo == GC_SPMM_ROW || algo == 0) {
    a.items = nullptr;
    a.n_items = n_rows;
  } else {
    set_error("%s: unknown algo %d", who, algo);
    return GC_ERR_VALUE;
  }
  GC_REQUIRE(a.ldb < (int64_t(1) << 30), GC_ERR_SHAPE, "%s: leading dimension too large", who);
  const int64_t K = a.K;
  if (a.flags & GC_SPMM_B_F16) {
    // fp16 operand rows: each lane gathers 16-byte chunks (8 columns = two
    // float4 slots), so the lane groups are half as wide as the fp32 shapes
    GC_REQUIRE(K % 8 == 0 && a.ldb % 8 == 0 && aligned16(a.B) && a.ldc % 4 == 0 &&
                   aligned16(a.C) && (a.partial == nullptr || aligned16(a.partial)),
               GC_ERR_UNSUPPORTED, "%s: fp16 operand needs K %% 8 == 0, ldb %% 8 == 0 and "
               "16-byte aligned B and C", who);
    GC_REQUIRE(!a.hints, GC_ERR_UNSUPPORTED, "%s: no hub tags with an fp16 operand", who);
    GC_REQUIRE(MODE == 0 || a.d_col != nullptr, GC_ERR_VALUE, "%s: fp16 rows need sigma", who);
    // chunked scales: one per 256-column pass (every fp16 shape above K = 256
    // runs 256 columns per pass); not for the SDDMM score (whole row per pass)
    GC_REQUIRE(a.sig_ld <= 1 || (MODE != 2 && a.d_col && K == (int64_t)a.sig_ld * 256),
               GC_ERR_UNSUPPORTED, "%s: %d scale chunks need K = %d (SpMM / GAT reassoc)", who,
               a.sig_ld, a.sig_ld * 256);
    GC_REQUIRE(MODE != 2 || (a.B_self != a.B && a.B_self != nullptr), GC_ERR_VALUE,
               "%s: fp16 rows need fp32 source rows B_self", who);
    cudaStream_t sth = as_stream(stream);
    const int sh = (int)((a.flags >> 8) & 3u);
    if (MODE == 2 && K > 512) return launch_cfg<32, 8, true, MODE, true>(a, sr, n_split, sth);
    if (MODE == 2 && K > 256) return launch_cfg<32, 4, true, MODE, true>(a, sr, n_split, sth);
    if (K <= 16) return launch_cfg<2, 2, true, MODE, true>(a, sr, n_split, sth);
    if (K <= 32) return sh ? launch_cfg<2, 4, true, MODE, true>(a, sr, n_split, sth)
                           : launch_cfg<4, 2, true, MODE, true>(a, sr, n_split, sth);
    if (K <= 64) return sh == 2 ? launch_cfg<2, 8, true, MODE, true>(a, sr, n_split, sth)
                      : sh == 1 ? launch_cfg<4, 4, true, MODE, true>(a, sr, n_split, sth)
                                : launch_cfg<8, 2, true, MODE, true>(a, sr, n_split, sth);
    if (K <= 128) return sh == 2 ? launch_cfg<4, 8, true, MODE, true>(a, sr, n_split, sth)
                       : sh == 1 ? launch_cfg<8, 4, true, MODE, true>(a, sr, n_split, sth)
                                 : launch_cfg<16, 2, true, MODE, true>(a, sr, n_split, sth);
    if (K <= 256) return sh == 2 ? launch_cfg<8, 8, true, MODE, true>(a, sr, n_split, sth)
                       : sh == 1 ? launch_cfg<16, 4, true, MODE, true>(a, sr, n_split, sth)
                                 : launch_cfg<32, 2, true, MODE, true>(a, sr, n_split, sth);
    return sh == 2 ? launch_cfg<8, 8, true, MODE, true>(a, sr, n_split, sth)
         : sh == 1 ? launch_cfg<16, 4, true, MODE, true>(a, sr, n_split, sth)
                   : launch_cfg<32, 2, true, MODE, true>(a, sr, n_split, sth);
  }
  const bool vec = (K % 4 == 0) && (a.ldb % 4 == 0) && (a.ldc % 4 == 0) && aligned16(a.B) &&
                   aligned16(a.C) && (a.partial == nullptr || aligned16(a.partial));
  if constexpr (MODE == 2) {
    GC_REQUIRE(vec && K <= 1024 && aligned16(a.a_src) && aligned16(a.a_dst), GC_ERR_UNSUPPORTED,
               "%s: needs K %% 4 == 0, K <= 1024 and 16-byte aligned operands", who);
    // the score needs the whole gathered row in one pass: wide rows get
    // 4 or 8 float4 slots per lane
    if (K > 512) return launch_cfg<32, 8, true, MODE>(a, sr, n_split, cudaStream_t(stream));
    if (K > 256) return launch_cfg<32, 4, true, MODE>(a, sr, n_split, cudaStream_t(stream));
  }
  cudaStream_t st = as_stream(stream);
  if (vec) {
    // lane-shrink s: LPR >> s lanes per row, each owning NV << s float4
    // columns (same columns per pass; more rows per warp for short rows)
    const int sh = (int)((a.flags >> 8) & 3u);
    if (K <= 8) return launch_cfg<2, 1, true, MODE>(a, sr, n_split, st);
    if (K <= 16) return sh ? launch_cfg<2, 2, true, MODE>(a, sr, n_split, st)
                           : launch_cfg<4, 1, true, MODE>(a, sr, n_split, st);
    if (K <= 32) return sh == 2 ? launch_cfg<2, 4, true, MODE>(a, sr, n_split, st)
                      : sh == 1 ? launch_cfg<4, 2, true, MODE>(a, sr, n_split, st)
                                : launch_cfg<8, 1, true, MODE>(a, sr, n_split, st);
    if (K <= 64) return sh == 2 ? launch_cfg<4, 4, true, MODE>(a, sr, n_split, st)
                      : sh == 1 ? launch_cfg<8, 2, true, MODE>(a, sr, n_split, st)
                                : launch_cfg<16, 1, true, MODE>(a, sr, n_split, st);
    if (K <= 128) return sh == 2 ? launch_cfg<8, 4, true, MODE>(a, sr, n_split, st)
                       : sh == 1 ? launch_cfg<16, 2, true, MODE>(a, sr, n_split, st)
                                 : launch_cfg<32, 1, true, MODE>(a, sr, n_split, st);
    return sh == 2 ? launch_cfg<8, 8, true, MODE>(a, sr, n_split, st)
         : sh == 1 ? launch_cfg<16, 4, true, MODE>(a, sr, n_split, st)
                   : launch_cfg<32, 2, true, MODE>(a, sr, n_split, st);
  }
  if (K <= 8) return launch_cfg<8, 1, false, MODE>(a, sr, n_split, st);
  if (K <= 16) return launch_cfg<16, 1, false, MODE>(a, sr, n_split, st);
  if (K <= 32) return launch_cfg<32, 1, false, MODE>(a, sr, n_split, st);
  if (K <= 64) return launch_cfg<32, 2, false, MODE>(a, sr, n_split, st);
  return launch_cfg<32, 4, false, MODE>(a, sr, n_split, st);
}

// Half-width gather operand (the TF32 class): with Y[j,:] = d[j] * X[j,:]
// (fp32; Y = X without d), e_j is chosen so that max_k |Y[j,k]| * 2^-e_j lies
// in [2^14, 2^15) and
//   Xh[j,k] = fp16_rn(Y[j,k] * 2^-e_j),   sigma[j] = 2^e_j,
// so X[j,:] * d[j] = sigma[j] * Xh[j,:] up to the fp16 rounding of each
// element (11 significant bits — the same input rounding TF32 applies).
// sigma stays a power of two (d folded into the values, as the GEMM epilogue
// folds its row scale), so unit-valued SpMM batches weigh their edges in fp16
// exactly (the fp16-weight FMA of spmm_kernel).
// A group of LPR lanes per row (LPR = K/4 up to 32: narrow rows do not leave
// lanes idle); each lane keeps its NC float4 chunks in registers between the
// max and the conversion, so the row is read once (K <= 4·LPR·NC, up to
// 4096), 8-byte writes.
// Optional projections (the GAT node scores, fused so the rows are read
// once): proj_out[p * n + r] = X[r,:] . P[p,:] for p < n_proj, in the same
// lane order and reduction tree as node_proj_kernel when LPR == 32.
template <int LPR, int NC>
__global__ void __launch_bounds__(256)
    pack_rows_f16_kernel(const float *__restrict__ X, int64_t ldx, int64_t n, int64_t K,
                         const float *__restrict__ d, __half *__restrict__ Xh, int64_t ldh,
                         float *__restrict__ sigma, bool vec, const float *__restrict__ P = nullptr,
                         int n_proj = 0, float *__restrict__ proj_out = nullptr) {
  const int gl = threadIdx.x % LPR;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR;
  const bool live = r < n;
  const float *x = X + (live ? r : 0) * ldx;
  float mx = 0.0f;
  const int64_t step = 4 * LPR;
  const float dr = (d && live) ? __ldg(d + r) : 1.0f;
  float4 v[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (vec && live) {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int64_t c = 4 * gl + i * step;
      if (c < K) {
        v[i] = ldg_f4(x + c);
        const float4 y = d ? make_float4(v[i].x * dr, v[i].y * dr, v[i].z * dr, v[i].w * dr) : v[i];
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(y.x), fabsf(y.y)), fmaxf(fabsf(y.z), fabsf(y.w))));
      }
    }
  } else if (live) {
    for (int64_t c = gl; c < K; c += LPR) mx = fmaxf(mx, fabsf(d ? __ldg(x + c) * dr : __ldg(x + c)));
  }
  mx = group_max<LPR>(mx);
  for (int q = 0; q < n_proj; ++q) {  // (vec only; warp-uniform loop)
    const float *pq = P + (int64_t)q * K;
    float acc = 0.0f;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int64_t c = 4 * gl + i * step;
      if (live && c < K) acc = fma4_dot(v[i], ldg_f4(pq + c), acc);
    }
    acc = group_sum<LPR>(acc);
    if (live && gl == 0) proj_out[(int64_t)q * n + r] = acc;
  }
  if (!live) return;
  // exponent of mx (exact): mx = m * 2^E, m in [1, 2)
  const int E = mx > 0.0f ? ((int)((__float_as_uint(mx) >> 23) & 0xff) - 127) : 0;
  const int e = mx > 0.0f && isfinite(mx) ? max(min(E - 14, 110), -110) : 0;
  const float down = __uint_as_float((uint32_t)(127 - e) << 23);  // 2^-e, |e| <= 110
  __half *h = Xh + r * ldh;
  if (vec) {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int64_t c = 4 * gl + i * step;
      if (c < K) {
        float4 y = v[i];
        if (d) y = make_float4(y.x * dr, y.y * dr, y.z * dr, y.w * dr);
        const __half2 a = __floats2half2_rn(y.x * down, y.y * down);
        const __half2 b = __floats2half2_rn(y.z * down, y.w * down);
        uint2 packed;
        packed.x = *reinterpret_cast<const uint32_t *>(&a);
        packed.y = *reinterpret_cast<const uint32_t *>(&b);
        *reinterpret_cast<uint2 *>(h + c) = packed;
      }
    }
  } else {
    for (int64_t c = gl; c < K; c += LPR)
      h[c] = __float2half_rn((d ? __ldg(x + c) * dr : __ldg(x + c)) * down);
  }
  if (gl == 0) sigma[r] = __uint_as_float((uint32_t)(127 + e) << 23);
}

__global__ void tag_hub_kernel(const int32_t *__restrict__ col, int64_t nnz,
                               const uint8_t *__restrict__ hot, int32_t *__restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = __ldg(col + p);
    out[p] = __ldg(hot + c) ? (int32_t)((uint32_t)c | 0x80000000u) : c;
  }
}

}  // namespace
}  // namespace gnnc

using namespace gnnc;

extern "C" int gc_pack_rows_f16_proj(const float *X, int64_t ldx, int64_t n_rows, int64_t K,
                                     const float *d, void *Xh, int64_t ldh, float *sigma,
                                     const float *P, int32_t n_proj, float *proj_out,
                                     void *stream);

extern "C" int gc_pack_rows_f16(const float *X, int64_t ldx, int64_t n_rows, int64_t K,
                                const float *d, void *Xh, int64_t ldh, float *sigma,
                                void *stream) {
  return gc_pack_rows_f16_proj(X, ldx, n_rows, K, d, Xh, ldh, sigma, nullptr, 0, nullptr, stream);
}

extern "C" int gc_pack_rows_f16_proj(const float *X, int64_t ldx, int64_t n_rows, int64_t K,
                                     const float *d, void *Xh, int64_t ldh, float *sigma,
                                     const float *P, int32_t n_proj, float *proj_out,
                                     void *stream) {
  GC_REQUIRE(n_rows >= 0 && K >= 0 && ldx >= K && ldh >= K, GC_ERR_SHAPE,
             "gc_pack_rows_f16: bad shape");
  GC_REQUIRE(n_proj >= 0 && n_proj <= 16 && (n_proj == 0 || (P && proj_out)), GC_ERR_VALUE,
             "gc_pack_rows_f16: projections need P and proj_out, n_proj <= 16");
  if (n_rows == 0) return GC_OK;
  GC_REQUIRE(X && Xh && sigma, GC_ERR_VALUE, "gc_pack_rows_f16: null operand");
  const bool vec = K % 4 == 0 && ldx % 4 == 0 && ldh % 4 == 0 && aligned16(X) &&
                   (reinterpret_cast<uintptr_t>(Xh) & 7u) == 0 && K <= 4096;
  GC_REQUIRE(n_proj == 0 || (vec && aligned16(P)), GC_ERR_UNSUPPORTED,
             "gc_pack_rows_f16: projections need the vectorised row layout (K %% 4 == 0, "
             "16-byte aligned X, P)");
  const int64_t q = vec ? (K + 3) / 4 : K;  // lanes a row could use
  const int lpr = q >= 32 ? 32 : q >= 16 ? 16 : q >= 8 ? 8 : q >= 4 ? 4 : q >= 2 ? 2 : 1;
  const int64_t chunks = vec ? (q + lpr - 1) / lpr : 1;  // float4 chunks per lane
  const int64_t blocks = (n_rows * lpr + 255) / 256;
  GC_REQUIRE(blocks < INT32_MAX, GC_ERR_SHAPE, "gc_pack_rows_f16: too many rows");
  __half *xh = static_cast<__half *>(Xh);
  cudaStream_t st = as_stream(stream);
#define GC_PACK(L, C)                                                                        \
  pack_rows_f16_kernel<L, C><<<(unsigned)blocks, 256, 0, st>>>(X, ldx, n_rows, K, d, xh, ldh, \
                                                              sigma, vec, P, n_proj, proj_out)
  // (below 32 lanes lpr is the largest power of two <= q, so a lane holds at
  // most two chunks)
  switch (lpr) {
    case 1: GC_PACK(1, 2); break;
    case 2: GC_PACK(2, 2); break;
    case 4: GC_PACK(4, 2); break;
    case 8: GC_PACK(8, 2); break;
    case 16: GC_PACK(16, 2); break;
    default:
      if (chunks <= 2) GC_PACK(32, 2);
      else if (chunks <= 4) GC_PACK(32, 4);
      else if (chunks <= 8) GC_PACK(32, 8);
      else GC_PACK(32, 32);
      break;
  }
#undef GC_PACK
  return check_launch("pack_rows_f16_kernel");
}

extern "C" int gc_tag_hub_columns(const int32_t *col_idx, int64_t nnz, const uint8_t *hot,
                                  int32_t *col_tagged, void *stream) {
  GC_REQUIRE(nnz >= 0, GC_ERR_SHAPE, "gc_tag_hub_columns: nnz < 0");
  if (nnz == 0) return GC_OK;
  GC_REQUIRE(col_idx && hot && col_tagged, GC_ERR_VALUE, "gc_tag_hub_columns: null operand");
  const int64_t blocks = std::min<int64_t>((nnz + 255) / 256, (int64_t)sm_count() * 32);
  tag_hub_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(col_idx, nnz, hot, col_tagged);
  return check_launch("tag_hub_kernel");
}

extern "C" int gc_spmm_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *values,
                           const float *d_row, const float *d_col, const float *B, int64_t ldb,
                           int64_t n_rows, int64_t n_cols, int64_t K, float *C, int64_t ldc,
                           uint32_t flags, int algo, const int32_t *items, int64_t n_items,
                           const int32_t *split_rows, int64_t n_split_rows, void *workspace,
                           size_t ws_bytes, void *stream) {
  GC_REQUIRE(n_rows >= 0 && n_cols >= 0 && K >= 0, GC_ERR_SHAPE, "gc_spmm_f32: negative size");
  GC_REQUIRE(ldb >= K && ldc >= K, GC_ERR_SHAPE, "gc_spmm_f32: leading dimension < K");
  GC_REQUIRE((flags & ~(GC_RELU | GC_ACCUMULATE | GC_HUB_TAGGED | GC_SPMM_SHRINK_MASK |
                         GC_SPMM_SIG_MASK |
                         GC_SPMM_B_F16)) == 0,
             GC_ERR_VALUE, "gc_spmm_f32: unknown flags 0x%x", flags);
  if (n_rows == 0 || K == 0) return GC_OK;
  GC_REQUIRE(row_ptr && C && (B || n_cols == 0), GC_ERR_VALUE, "gc_spmm_f32: null operand");
  GC_REQUIRE(n_rows < INT32_MAX && n_cols < INT32_MAX, GC_ERR_SHAPE,
             "gc_spmm_f32: int32 index range exceeded");
  SpmmArgs a{};
  a.row_ptr = row_ptr;
  a.col_idx = col_idx;
  a.values = values;
  a.d_row = d_row;
  a.d_col = d_col;
  a.B = B;
  a.ldb = ldb;
  a.K = K;
  a.C = C;
  a.ldc = ldc;
  a.flags = flags & ~GC_SPMM_SIG_MASK;
  a.sig_ld = (int)((flags & GC_SPMM_SIG_MASK) >> 12) + 1;
  a.hints = (flags & GC_HUB_TAGGED) != 0;
  return dispatch<0>(a, n_rows, algo, items, n_items, split_rows, n_split_rows, workspace,
                         ws_bytes, stream, "gc_spmm_f32");
}

// ---------------------------------------------------------------------------
// Aggregate-first layer with a narrow update fused into the epilogue (SURVEY
// N4, reference gcn.py:119-122 `gemm(spmm(a, h), w)`): C = epi(D_row A D_col
// B) W for K1 <= 256, K2 <= 32 — the n x K1 aggregate never leaves
// registers.  One lane group per row (LPR = K1/4 up to 32 lanes, NV float4
// slots each, one column pass), edges in order (the aggregate is the SpMM's
// own sum, bit for bit), then per output column c a lane-partial dot with
// W[:, c] (W^T staged in shared memory, read as float4) and a group sum.
template <int LPR, int NV>
__global__ void __launch_bounds__(kThreads)
    spmm_w_kernel(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                  const float *__restrict__ values, const float *__restrict__ d_row,
                  const float *__restrict__ d_col, const float *__restrict__ B, int64_t ldb,
                  int K1, const float *__restrict__ W, int K2, float *__restrict__ C,
                  int64_t ldc, int64_t n_rows, uint32_t flags) {
  constexpr int U = LPR < 4 ? LPR : 4;
  constexpr int K1P = LPR * NV * 4;  // padded row width (one pass)
  extern __shared__ __align__(16) float wt_smem[];  // [K2][K1P]: W^T, zero padded
  for (int i = threadIdx.x; i < K2 * K1P; i += kThreads) {
    const int c = i / K1P, k = i % K1P;
    wt_smem[i] = k < K1 ? __ldg(W + (int64_t)k * K2 + c) : 0.0f;
  }
  __syncthreads();
  const int gl = threadIdx.x % LPR;
  bool colok[NV];
  int coff[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    coff[v] = v * LPR * 4 + gl * 4;
    colok[v] = coff[v] < K1;
  }
  const float4 *wt4 = reinterpret_cast<const float4 *>(wt_smem);
  // grid-stride over row groups: W^T is staged once per CTA
  for (int64_t row = ((int64_t)blockIdx.x * kThreads + threadIdx.x) / LPR; ;
       row += (int64_t)gridDim.x * (kThreads / LPR)) {
    const int64_t first = row - (int64_t)(threadIdx.x / LPR);  // warp-uniform exit test
    if (__shfl_sync(0xffffffffu, (int)(first >= n_rows), 0)) break;
    const bool live = row < n_rows;
    int beg = 0, end = 0;
    if (live) {
      beg = __ldg(row_ptr + row);
      end = __ldg(row_ptr + row + 1);
    }
    float4 acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int len = end - beg;
    const int wmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)len);
    for (int base = 0; base < wmax; base += LPR) {
      int j = 0;
      float w = 0.0f;  // lanes past the row's end: row 0 with weight 0
      if (base + gl < len) {
        j = ldg_stream_i32(col_idx + beg + base + gl);
        w = values ? ldg_stream_f32(values + beg + base + gl) : 1.0f;
        if (d_col) w *= __ldg(d_col + j);
      }
      const int cntw = min(LPR, wmax - base);
#pragma unroll 1
      for (int e0 = 0; e0 < cntw; e0 += U) {
        float4 bv[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int je = __shfl_sync(0xffffffffu, j, e0 + u, LPR);
          const float *brow = B + (int64_t)je * ldb;
#pragma unroll
          for (int v = 0; v < NV; ++v)
            if (colok[v]) bv[u][v] = ldg_f4(brow + coff[v]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float we = __shfl_sync(0xffffffffu, w, e0 + u, LPR);
          if (base + e0 + u < len) {
#pragma unroll
            for (int v = 0; v < NV; ++v)
              if (colok[v]) fma_into(acc[v], we, bv[u][v]);
          }
        }
      }
    }
    const float ds = (live && d_row) ? __ldg(d_row + row) : 1.0f;
    for (int c = 0; c < K2; ++c) {
      float part = 0.0f;
#pragma unroll
      for (int v = 0; v < NV; ++v) part += dot_of(acc[v], wt4[(c * K1P + coff[v]) / 4]);
      part = group_sum<LPR>(part);
      if (live && gl == c % LPR) {
        float o = part * ds;
        if (flags & GC_RELU) o = fmaxf(o, 0.0f);
        C[row * ldc + c] = o;
      }
    }
  }
}

template <int LPR, int NV>
int launch_spmm_w(const int32_t *row_ptr, const int32_t *col_idx, const float *values,
                  const float *d_row, const float *d_col, const float *B, int64_t ldb, int K1,
                  const float *W, int K2, float *C, int64_t ldc, int64_t n_rows, uint32_t flags,
                  cudaStream_t st) {
  const int smem = K2 * LPR * NV * 4 * (int)sizeof(float);
  const int64_t groups_per_block = kThreads / LPR;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // enough CTAs to fill the SMs (W^T staged once per CTA), never more than rows
  const int64_t need = (n_rows + groups_per_block - 1) / groups_per_block;
  const unsigned grid = (unsigned)std::min<int64_t>(need, (int64_t)sms * 8);
  spmm_w_kernel<LPR, NV><<<grid, kThreads, smem, st>>>(row_ptr, col_idx, values, d_row, d_col, B,
                                                       ldb, K1, W, K2, C, ldc, n_rows, flags);
  return check_launch("spmm_w_kernel");
}

extern "C" int gc_spmm_gemm_f32(const int32_t *row_ptr, const int32_t *col_idx,
                                const float *values, const float *d_row, const float *d_col,
                                const float *B, int64_t ldb, int64_t n_rows, int64_t n_cols,
                                int64_t K1, const float *W, int64_t K2, float *C, int64_t ldc,
                                uint32_t flags, void *stream) {
  GC_REQUIRE(n_rows >= 0 && n_cols >= 0 && K1 >= 0 && K2 >= 0, GC_ERR_SHAPE,
             "gc_spmm_gemm_f32: negative size");
  GC_REQUIRE((flags & ~GC_RELU) == 0, GC_ERR_VALUE, "gc_spmm_gemm_f32: unknown flags 0x%x", flags);
  GC_REQUIRE(K1 % 4 == 0 && K1 <= 256 && K2 <= 32, GC_ERR_UNSUPPORTED,
             "gc_spmm_gemm_f32: needs K1 %% 4 == 0, K1 <= 256 and K2 <= 32 (K1=%lld, K2=%lld)",
             (long long)K1, (long long)K2);
  GC_REQUIRE(ldb >= K1 && ldb % 4 == 0 && ldc >= K2, GC_ERR_SHAPE,
             "gc_spmm_gemm_f32: ldb must be >= K1 and a multiple of 4, ldc >= K2");
  if (n_rows == 0 || K2 == 0) return GC_OK;
  GC_REQUIRE(row_ptr && C && W && (B || n_cols == 0) && aligned16(B), GC_ERR_VALUE,
             "gc_spmm_gemm_f32: null or misaligned operand");
  GC_REQUIRE(n_rows < INT32_MAX && n_cols < INT32_MAX, GC_ERR_SHAPE,
             "gc_spmm_gemm_f32: int32 index range exceeded");
  cudaStream_t st = as_stream(stream);
  const int k1 = (int)K1, k2 = (int)K2;
  if (K1 <= 8) return launch_spmm_w<2, 1>(row_ptr, col_idx, values, d_row, d_col, B, ldb, k1, W, k2, C, ldc, n_rows, flags, st);
  if (K1 <= 16) return launch_spmm_w<4, 1>(row_ptr, col_idx, values, d_row, d_col, B, ldb, k1, W, k2, C, ldc, n_rows, flags, st);
  if (K1 <= 32) return launch_spmm_w<8, 1>(row_ptr, col_idx, values, d_row, d_col, B, ldb, k1, W, k2, C, ldc, n_rows, flags, st);
  if (K1 <= 64) return launch_spmm_w<16, 1>(row_ptr, col_idx, values, d_row, d_col, B, ldb, k1, W, k2, C, ldc, n_rows, flags, st);
  if (K1 <= 128) return launch_spmm_w<32, 1>(row_ptr, col_idx, values, d_row, d_col, B, ldb, k1, W, k2, C, ldc, n_rows, flags, st);
  return launch_spmm_w<32, 2>(row_ptr, col_idx, values, d_row, d_col, B, ldb, k1, W, k2, C, ldc, n_rows, flags, st);
}

extern "C" int gc_gat_sddmm_aggregate_f32(const int32_t *row_ptr, const int32_t *col_idx,
                                          const float *a_src, const float *a_dst, float slope,
                                          const float *B, int64_t ldb, const float *B_self,
                                          int64_t ld_self, const float *sigma, int64_t n_rows,
                                          int64_t K,
                                          float *C, int64_t ldc, uint32_t flags, int algo,
                                          const int32_t *items, int64_t n_items,
                                          const int32_t *split_rows, int64_t n_split_rows,
                                          void *workspace, size_t ws_bytes, void *stream) {
  GC_REQUIRE(n_rows >= 0 && K >= 1, GC_ERR_SHAPE, "gc_gat_sddmm_aggregate_f32: bad size");
  GC_REQUIRE(ldb >= K && ldc >= K, GC_ERR_SHAPE,
             "gc_gat_sddmm_aggregate_f32: leading dimension < K");
  GC_REQUIRE((flags & ~(GC_RELU | GC_HUB_TAGGED | GC_SPMM_SHRINK_MASK | GC_SPMM_B_F16 |
                         GC_SPMM_SIG_MASK)) == 0,
             GC_ERR_VALUE, "gc_gat_sddmm_aggregate_f32: unknown flags 0x%x", flags);
  GC_REQUIRE(slope > 0.0f && slope < 1.0f, GC_ERR_VALUE,
             "gc_gat_sddmm_aggregate_f32: leaky_slope must lie in (0, 1)");
  if (n_rows == 0) return GC_OK;
  GC_REQUIRE(row_ptr && C && B && a_src && a_dst, GC_ERR_VALUE,
             "gc_gat_sddmm_aggregate_f32: null operand");
  GC_REQUIRE(n_rows < INT32_MAX, GC_ERR_SHAPE, "gc_gat_sddmm_aggregate_f32: int32 range");
  GC_REQUIRE(B_self == nullptr || (ld_self >= K && ld_self % 4 == 0 && aligned16(B_self)),
             GC_ERR_UNSUPPORTED, "gc_gat_sddmm_aggregate_f32: B_self needs ld >= K, ld %% 4 == 0 "
             "and 16-byte alignment");
  SpmmArgs a{};
  a.row_ptr = row_ptr;
  a.col_idx = col_idx;
  a.B = B;
  a.ldb = ldb;
  a.B_self = B_self ? B_self : B;
  a.ld_self = B_self ? ld_self : ldb;
  a.d_col = sigma;  // GC_SPMM_B_F16: per-row scales of the fp16 rows
  a.K = K;
  a.C = C;
  a.ldc = ldc;
  a.flags = flags & ~GC_SPMM_SIG_MASK;
  a.sig_ld = (int)((flags & GC_SPMM_SIG_MASK) >> 12) + 1;
  a.hints = (flags & GC_HUB_TAGGED) != 0;
  a.a_src = a_src;
  a.a_dst = a_dst;
  a.slope = slope;
  return dispatch<2>(a, n_rows, algo, items, n_items, split_rows, n_split_rows, workspace,
                     ws_bytes, stream, "gc_gat_sddmm_aggregate_f32");
}

extern "C" int gc_gat_aggregate_f32(const int32_t *row_ptr, const int32_t *col_idx,
                                    const float *s, const float *t, float slope, const float *B,
                                    int64_t ldb, const float *sigma, int64_t n_rows, int64_t n_cols,
                                    int64_t K,
                                    float *C, int64_t ldc, uint32_t flags, int algo,
                                    const int32_t *items, int64_t n_items,
                                    const int32_t *split_rows, int64_t n_split_rows,
                                    void *workspace, size_t ws_bytes, void *stream) {
  GC_REQUIRE(n_rows >= 0 && n_cols >= 0 && K >= 0, GC_ERR_SHAPE,
             "gc_gat_aggregate_f32: negative size");
  GC_REQUIRE(ldb >= K && ldc >= K, GC_ERR_SHAPE, "gc_gat_aggregate_f32: leading dimension < K");
  GC_REQUIRE((flags & ~(GC_RELU | GC_HUB_TAGGED | GC_SPMM_SHRINK_MASK | GC_SPMM_B_F16 |
                         GC_SPMM_SIG_MASK)) == 0,
             GC_ERR_VALUE, "gc_gat_aggregate_f32: unknown flags 0x%x", flags);
  GC_REQUIRE(slope > 0.0f && slope < 1.0f, GC_ERR_VALUE,
             "gc_gat_aggregate_f32: leaky_slope must lie in (0, 1)");
  if (n_rows == 0 || K == 0) return GC_OK;
  GC_REQUIRE(row_ptr && C && s && t && (B || n_cols == 0), GC_ERR_VALUE,
             "gc_gat_aggregate_f32: null operand");
  GC_REQUIRE(n_rows < INT32_MAX && n_cols < INT32_MAX, GC_ERR_SHAPE,
             "gc_gat_aggregate_f32: int32 index range exceeded");
  SpmmArgs a{};
  a.row_ptr = row_ptr;
  a.col_idx = col_idx;
  a.B = B;
  a.ldb = ldb;
  a.K = K;
  a.C = C;
  a.ldc = ldc;
  a.flags = flags & ~GC_SPMM_SIG_MASK;
  a.sig_ld = (int)((flags & GC_SPMM_SIG_MASK) >> 12) + 1;
  a.hints = (flags & GC_HUB_TAGGED) != 0;
  a.s = s;
  a.t = t;
  a.slope = slope;
  a.d_col = sigma;  // GC_SPMM_B_F16: per-row scales of the fp16 rows
  return dispatch<1>(a, n_rows, algo, items, n_items, split_rows, n_split_rows, workspace,
                        ws_bytes, stream, "gc_gat_aggregate_f32");
}
