// Edge-wise kernels over the CSR pattern: SDDMM (sparse.py:222-232), the k=1
// normalisation SDDMM (gcn.py:103-112) and the GAT attention in both
// compositions (gat.py:72-114): the reassociated per-node projections + fused
// LeakyReLU/edge-softmax, and the SDDMM-over-edges variant.
//
// All of these are HBM-bound streams over col_idx (+ values) with an L2-resident
// per-node gather (d, t); each row is owned by one lane group, the reductions
// use a fixed shuffle tree, so results are deterministic.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace gnnc {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxHeads = 8;

// ---------------------------------------------------------------------------
// generic SDDMM: out[p] = a[p] * sum_t B[i,t] * Cm[j,t]  (t ascending per edge,
// one lane per edge, exactly the reference's loop order)
// ---------------------------------------------------------------------------
template <int LPR>
__global__ void __launch_bounds__(kThreads)
    sddmm_kernel(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                 const float *__restrict__ a_vals, const float *__restrict__ B, int64_t ldb,
                 const float *__restrict__ Cm, int64_t ldc, int64_t n_rows, int64_t k,
                 float *__restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * (kThreads / LPR) + threadIdx.x / LPR;
  const int gl = threadIdx.x % LPR;
  if (row >= n_rows) return;
  const int beg = row_ptr[row], end = row_ptr[row + 1];
  const float *bi = B + row * ldb;
  for (int p = beg + gl; p < end; p += LPR) {
    const float *cj = Cm + (int64_t)ldg_stream_i32(col_idx + p) * ldc;
    float acc = 0.0f;
    for (int64_t t = 0; t < k; ++t) acc = fmaf(__ldg(bi + t), __ldg(cj + t), acc);
    out[p] = (a_vals ? ldg_stream_f32(a_vals + p) : 1.0f) * acc;
  }
}

// k = 1 normalisation: out[p] = a[p] * (d[i] * d[j]).  Edge-parallel: each
// warp owns a fixed chunk of edges (uniform work on power-law graphs, whose
// hub rows would otherwise serialise one warp each), finds the chunk's first
// row by binary search in row_ptr, and each lane walks rows as it strides.
__device__ __forceinline__ int64_t row_of_edge(const int32_t *__restrict__ row_ptr,
                                               int64_t n_rows, int64_t p) {
  int64_t lo = 0, hi = n_rows;  // last r with row_ptr[r] <= p (skips empty rows)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)__ldg(row_ptr + mid) <= p) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Rows of a step's 32 consecutive edges: lane k holds the end of row
// r0 + k (row_ptr[r0 + 1 + k]); an edge's row offset is the number of those
// ends <= its index, found by a 5-step binary search over the lanes with
// shuffles — no dependent global loads per row crossing.  Returns 32 when
// the 32-row window does not reach the edge (runs of empty rows).
__device__ __forceinline__ int row_offset_in_window(int bk, int p) {
  int cnt = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const int b = __shfl_sync(0xffffffffu, bk, cnt + step - 1);
    if (b <= p) cnt += step;
  }
  const int b31 = __shfl_sync(0xffffffffu, bk, 31);  // (all lanes: full-mask shuffle)
  if (cnt == 31 && b31 <= p) cnt = 32;  // the window ends before p: caller walks on
  return cnt;
}

// LONG (mean degree >= 128): a step that stays inside the current row skips
// the window (most steps on dense graphs); short rows always search.
template <bool LONG>
__global__ void __launch_bounds__(kThreads)
    sddmm_norm_kernel(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                      const float *__restrict__ a_vals, const float *__restrict__ d,
                      int64_t n_rows, int64_t nnz, int64_t chunk, float *__restrict__ out) {
  const int64_t w = ((int64_t)blockIdx.x * kThreads + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int64_t p0 = w * chunk;
  if (p0 >= nnz) return;
  const int64_t p1 = min(nnz, p0 + chunk);
  int64_t r0 = row_of_edge(row_ptr, n_rows, p0);  // warp-uniform search, once per chunk
  int64_t rend0 = __ldg(row_ptr + r0 + 1);          // end of row r0 (warp-uniform)
  for (int64_t base = p0; base < p1; base += 32) {
    const int64_t p = base + lane;
    const bool ok = p < p1;
    const int j = ok ? ldg_stream_i32(col_idx + p) : 0;
    const float av = (a_vals && ok) ? ldg_stream_f32(a_vals + p) : 1.0f;
    int64_t row = r0;
    if (!LONG || min(base + 31, p1 - 1) >= rend0) {  // the step crosses a row end (warp-uniform)
      const int64_t rk = r0 + 1 + lane;
      const int bk = rk <= n_rows ? __ldg(row_ptr + rk) : INT32_MAX;
      const int64_t pc = min(p, p1 - 1);  // idle lanes take the last edge's row
      const int off = row_offset_in_window(bk, (int)pc);
      row = r0 + off;
      if (off == 32) {  // > 31 row ends within the step (runs of empty rows): walk
        int64_t rend = __ldg(row_ptr + row + 1);
        while (pc >= rend) rend = __ldg(row_ptr + (++row) + 1);
      }
      const int off31 = __shfl_sync(0xffffffffu, off, 31);
      r0 = __shfl_sync(0xffffffffu, row, 31);  // row of the step's last edge
      const int be = __shfl_sync(0xffffffffu, bk, off31 & 31);
      rend0 = off31 < 32 ? be : __ldg(row_ptr + r0 + 1);
    }
    if (ok) out[p] = av * (__ldg(d + row) * __ldg(d + j));
  }
}

// ---------------------------------------------------------------------------
// node projections s = HW·a_src, t = HW·a_dst per head (warp per row)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
    node_proj_kernel(const float *__restrict__ HW, int64_t ld, int64_t n_rows, int64_t k2,
                     int heads, int64_t head_stride, const float *__restrict__ a_src,
                     const float *__restrict__ a_dst, float *__restrict__ s,
                     float *__restrict__ t, bool vec) {
  const int64_t row = (int64_t)blockIdx.x * (kThreads / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= n_rows) return;
  const float *hr = HW + row * ld;
  if (vec && head_stride == 0 && k2 <= 1024) {
    // every head projects the same row (the folded-vector scores s = H (W a)):
    // the row is read once into registers, all loads in flight together; the
    // per-head sums keep the loop's order, so results are unchanged
    float4 xv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t c = 4 * lane + 128 * i;
      xv[i] = c < k2 ? ldg_f4(hr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int h = 0; h < heads; ++h) {
      const float *al = a_src + (int64_t)h * k2;
      const float *ar = a_dst + (int64_t)h * k2;
      float ss = 0.f, tt = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t c = 4 * lane + 128 * i;
        if (c < k2) {
          ss = fma4_dot(xv[i], ldg_f4(al + c), ss);
          tt = fma4_dot(xv[i], ldg_f4(ar + c), tt);
        }
      }
      ss = group_sum<32>(ss);
      tt = group_sum<32>(tt);
      if (lane == 0) {
        s[(int64_t)h * n_rows + row] = ss;
        if (t) t[(int64_t)h * n_rows + row] = tt;
      }
    }
    return;
  }
  for (int h = 0; h < heads; ++h) {
    const float *x = hr + (int64_t)h * head_stride;
    const float *al = a_src + (int64_t)h * k2;
    const float *ar = a_dst + (int64_t)h * k2;
    float ss = 0.f, tt = 0.f;
    if (vec) {
      for (int64_t c = 4 * lane; c < k2; c += 128) {
        const float4 xv = ldg_f4(x + c);
        ss = fma4_dot(xv, ldg_f4(al + c), ss);
        tt = fma4_dot(xv, ldg_f4(ar + c), tt);
      }
    } else {
      for (int64_t c = lane; c < k2; c += 32) {
        const float xv = __ldg(x + c);
        ss = fmaf(xv, __ldg(al + c), ss);
        tt = fmaf(xv, __ldg(ar + c), tt);
      }
    }
    ss = group_sum<32>(ss);
    tt = group_sum<32>(tt);
    if (lane == 0) {
      s[(int64_t)h * n_rows + row] = ss;
      if (t) t[(int64_t)h * n_rows + row] = tt;
    }
  }
}

// ---------------------------------------------------------------------------
// fused LeakyReLU + edge softmax (reassociated attention), multi-head.
// Pass 1: per-lane online (max, sum); group merge.  Pass 2: normalised write.
// EGIVEN: the scores were staged in `alpha` by attn_score_kernel (SDDMM form)
// and are normalised in place.
// ---------------------------------------------------------------------------
// One heavy row per CTA (power-law hubs): kThreads lanes stride the row, the
// (max, sum) pairs merge through a fixed shuffle tree and then across warps in
// warp order, so the result stays deterministic.
template <bool EGIVEN>
__device__ __forceinline__ void softmax_row_cta(int64_t row, const int32_t *__restrict__ row_ptr,
                                                const int32_t *__restrict__ col_idx,
                                                const float *__restrict__ s,
                                                const float *__restrict__ t, int heads,
                                                float slope, int64_t n_rows, int64_t nnz,
                                                float *__restrict__ alpha) {
  __shared__ float red_m[kThreads / 32][kMaxHeads], red_z[kThreads / 32][kMaxHeads];
  __shared__ float fin_m[kMaxHeads], fin_z[kMaxHeads];
  const int beg = row_ptr[row], end = row_ptr[row + 1];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float si[kMaxHeads], m[kMaxHeads], z[kMaxHeads];
#pragma unroll
  for (int h = 0; h < kMaxHeads; ++h) {
    si[h] = (!EGIVEN && h < heads) ? __ldg(s + (int64_t)h * n_rows + row) : 0.f;
    m[h] = -INFINITY;
    z[h] = 0.f;
  }
  for (int p = beg + threadIdx.x; p < end; p += kThreads) {
    const int j = EGIVEN ? 0 : __ldg(col_idx + p);
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
      if (h >= heads) break;
      const float e = EGIVEN ? alpha[(int64_t)h * nnz + p]
                             : leaky(si[h] + __ldg(t + (int64_t)h * n_rows + j), slope);
      if (e > m[h]) {
        z[h] = z[h] * __expf(m[h] - e) + 1.0f;
        m[h] = e;
      } else {
        z[h] += __expf(e - m[h]);
      }
    }
  }
#pragma unroll
  for (int h = 0; h < kMaxHeads; ++h) {
    if (h >= heads) break;
    const float mg = group_max<32>(m[h]);
    const float zl = (m[h] == -INFINITY) ? 0.f : z[h] * __expf(m[h] - mg);
    const float zg = group_sum<32>(zl);
    if (lane == 0) red_m[warp][h] = mg, red_z[warp][h] = zg;
  }
  __syncthreads();
  if (threadIdx.x < heads) {
    const int h = threadIdx.x;
    float mm = -INFINITY;
    for (int w = 0; w < kThreads / 32; ++w) mm = fmaxf(mm, red_m[w][h]);
    float zz = 0.f;
    for (int w = 0; w < kThreads / 32; ++w)
      if (red_m[w][h] != -INFINITY) zz += red_z[w][h] * __expf(red_m[w][h] - mm);
    fin_m[h] = mm;
    fin_z[h] = 1.0f / zz;  // reciprocal: one multiply per edge below
  }
  __syncthreads();
  for (int p = beg + threadIdx.x; p < end; p += kThreads) {
    const int j = EGIVEN ? 0 : __ldg(col_idx + p);
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
      if (h >= heads) break;
      const float e = EGIVEN ? alpha[(int64_t)h * nnz + p]
                             : leaky(si[h] + __ldg(t + (int64_t)h * n_rows + j), slope);
      alpha[(int64_t)h * nnz + p] = __expf(e - fin_m[h]) * fin_z[h];
    }
  }
}

// Blocks [0, n_heavy) take one heavy row each (rows longer than `th`, listed
// by the caller); the remaining blocks give every other row a group of LPR
// lanes.  Without a heavy list every row goes to the lane groups.
template <int LPR, bool EGIVEN>
__global__ void __launch_bounds__(kThreads)
    edge_softmax_kernel(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                        const float *__restrict__ s, const float *__restrict__ t, int heads,
                        float slope, int64_t n_rows, int64_t nnz,
                        const int32_t *__restrict__ heavy, int64_t n_heavy, int th,
                        float *__restrict__ alpha) {
  if ((int64_t)blockIdx.x < n_heavy) {
    softmax_row_cta<EGIVEN>(heavy[blockIdx.x], row_ptr, col_idx, s, t, heads, slope, n_rows, nnz,
                            alpha);
    return;
  }
  const int64_t row = ((int64_t)blockIdx.x - n_heavy) * (kThreads / LPR) + threadIdx.x / LPR;
  const int gl = threadIdx.x % LPR;
  bool live = row < n_rows;
  int beg = live ? row_ptr[row] : 0, end = live ? row_ptr[row + 1] : 0;
  if (heavy && end - beg > th) live = false, beg = end = 0;  // owned by a CTA above
  float si[kMaxHeads], m[kMaxHeads], z[kMaxHeads];
#pragma unroll
  for (int h = 0; h < kMaxHeads; ++h) {
    si[h] = (!EGIVEN && live && h < heads) ? __ldg(s + (int64_t)h * n_rows + row) : 0.f;
    m[h] = -INFINITY;
    z[h] = 0.f;
  }
  // The lane's first CE edges keep their column and head-0 score in
  // registers (unrolled: no local-memory indexing), so pass 2 re-gathers
  // nothing for rows of <= CE * LPR edges — the dependent col -> t_j load
  // pair was the kernel's latency chain.
  constexpr int CE = 4;
  int jc[CE];
  float ec[CE];
  auto score = [&](int h, int p, int j) {
    return EGIVEN ? alpha[(int64_t)h * nnz + p]
                  : leaky(si[h] + __ldg(t + (int64_t)h * n_rows + j), slope);
  };
  auto update = [&](int h, float e) {
    if (e > m[h]) {
      z[h] = z[h] * __expf(m[h] - e) + 1.0f;
      m[h] = e;
    } else {
      z[h] += __expf(e - m[h]);
    }
  };
#pragma unroll
  for (int k = 0; k < CE; ++k) {
    const int p = beg + gl + k * LPR;
    jc[k] = 0;
    ec[k] = 0.f;
    if (p < end) {
      const int j = EGIVEN ? 0 : __ldg(col_idx + p);
      jc[k] = j;
#pragma unroll
      for (int h = 0; h < kMaxHeads; ++h) {
        if (h >= heads) break;
        const float e = score(h, p, j);
        if (h == 0) ec[k] = e;
        update(h, e);
      }
    }
  }
  for (int p = beg + gl + CE * LPR; p < end; p += LPR) {
    const int j = EGIVEN ? 0 : __ldg(col_idx + p);
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
      if (h >= heads) break;
      update(h, score(h, p, j));
    }
  }
  float inv[kMaxHeads];
#pragma unroll
  for (int h = 0; h < kMaxHeads; ++h) {
    inv[h] = 0.f;
    if (h >= heads) break;
    const float mg = group_max<LPR>(m[h]);
    const float zl = (m[h] == -INFINITY) ? 0.f : z[h] * __expf(m[h] - mg);
    z[h] = group_sum<LPR>(zl);
    m[h] = mg;
    inv[h] = 1.0f / z[h];
  }
  if (!live || end == beg) return;
#pragma unroll
  for (int k = 0; k < CE; ++k) {
    const int p = beg + gl + k * LPR;
    if (p < end) {
#pragma unroll
      for (int h = 0; h < kMaxHeads; ++h) {
        if (h >= heads) break;
        const float e = h == 0 ? ec[k] : score(h, p, jc[k]);
        alpha[(int64_t)h * nnz + p] = __expf(e - m[h]) * inv[h];
      }
    }
  }
  for (int p = beg + gl + CE * LPR; p < end; p += LPR) {
    const int j = EGIVEN ? 0 : __ldg(col_idx + p);
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
      if (h >= heads) break;
      alpha[(int64_t)h * nnz + p] = __expf(score(h, p, j) - m[h]) * inv[h];
    }
  }
}

// lanes per row and the heavy-row threshold, both from the mean degree
// (exported as gc_edge_softmax_heavy_threshold so the caller can list the
// heavy rows once per pattern)
inline int softmax_lpr(int64_t n_rows, int64_t nnz) {
  const double avg = (double)nnz / (double)(n_rows > 0 ? n_rows : 1);
  return avg <= 12.0 ? 8 : avg <= 64.0 ? 16 : 32;
}
inline int softmax_th(int64_t n_rows, int64_t nnz) { return 16 * softmax_lpr(n_rows, nnz); }

template <bool EGIVEN>
int launch_softmax(const int32_t *row_ptr, const int32_t *col_idx, const float *s, const float *t,
                   int heads, float slope, int64_t n_rows, int64_t nnz, const int32_t *heavy,
                   int64_t n_heavy, float *alpha, cudaStream_t st) {
  const int lpr = softmax_lpr(n_rows, nnz);
  const int th = softmax_th(n_rows, nnz);
  if (!heavy) n_heavy = 0;
  const int64_t light = (n_rows + (kThreads / lpr) - 1) / (kThreads / lpr);
  const int64_t blocks = light + n_heavy;
  if (blocks >= INT32_MAX) {
    set_error("edge softmax: row count %lld too large", (long long)n_rows);
    return GC_ERR_SHAPE;
  }
  if (lpr == 8)
    edge_softmax_kernel<8, EGIVEN><<<(unsigned)blocks, kThreads, 0, st>>>(
        row_ptr, col_idx, s, t, heads, slope, n_rows, nnz, heavy, n_heavy, th, alpha);
  else if (lpr == 16)
    edge_softmax_kernel<16, EGIVEN><<<(unsigned)blocks, kThreads, 0, st>>>(
        row_ptr, col_idx, s, t, heads, slope, n_rows, nnz, heavy, n_heavy, th, alpha);
  else
    edge_softmax_kernel<32, EGIVEN><<<(unsigned)blocks, kThreads, 0, st>>>(
        row_ptr, col_idx, s, t, heads, slope, n_rows, nnz, heavy, n_heavy, th, alpha);
  return check_launch("edge_softmax_kernel");
}

// ---------------------------------------------------------------------------
// attention as an SDDMM over edges:
//   e_p = LeakyReLU(a_src·HW_i + a_dst·HW_j)  for every edge p = (i, j),
// the k2-wide target dot product gathered per edge (cost m·2k2), then the
// same max-shifted row softmax as the reassociated form.
// Stage 1 (attn_score_kernel) is edge-parallel: each lane group owns a fixed
// chunk of edges (uniform work whatever the row lengths — power-law rows no
// longer serialise one warp), finds its first row by binary search in
// row_ptr and walks rows as the chunk advances; U edges are gathered at once.
// The source term a_src·HW_i is one k2-wide dot per node (node_proj_kernel).
// Stage 2 (edge_softmax_kernel<.., true>) normalises the staged scores in
// place, row by row.
// ---------------------------------------------------------------------------
template <int LPR, int NV, int U, bool VEC>
__global__ void __launch_bounds__(kThreads)
    attn_score_kernel(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                      const float *__restrict__ HW, int64_t ld, int64_t k2, int heads,
                      const float *__restrict__ s, const float *__restrict__ a_dst, float slope,
                      int64_t n_rows, int64_t nnz, int64_t chunk, float *__restrict__ e_out) {
  // Edges are taken in batches of LPR: lane gl loads batch edge gl's column
  // (coalesced) and walks its own row index forward; the next batch's
  // columns are in flight while the current batch is gathered U edges at a
  // time.  Lane gl owns column slots c0 + W*(gl + LPR*v), v < NV (W = 4
  // floats when VEC), so all U*NV gathers of a step are issued before the
  // first FMA and each per-edge dot is reduced over only LPR lanes.
  constexpr int W = VEC ? 4 : 1;
  constexpr int PASS = W * LPR * NV;
  const int gl = threadIdx.x % LPR;
  const int64_t grp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) / LPR;
  const int64_t p0 = grp * chunk;
  if (p0 >= nnz) return;  // group-uniform
  const int64_t p1 = min(nnz, p0 + chunk);
  int64_t row = row_of_edge(row_ptr, n_rows, p0);  // this lane's row, walked forward
  int64_t rend = __ldg(row_ptr + row + 1);
  int jc = (p0 + gl < p1) ? ldg_stream_i32(col_idx + p0 + gl) : 0;
  for (int64_t b = p0; b < p1; b += LPR) {
    const int jn = (b + LPR + gl < p1) ? ldg_stream_i32(col_idx + b + LPR + gl) : 0;
    const int64_t pe = b + gl;
    if (pe < p1)
      while (pe >= rend) rend = __ldg(row_ptr + (++row) + 1);
    const int rc = (int)row;
    const int cnt = (int)min((int64_t)LPR, p1 - b);
#pragma unroll 1
    for (int e0 = 0; e0 < cnt; e0 += U) {
      const float *hj[U];
      int ru[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int src = (e0 + u) & (LPR - 1);
        ok[u] = e0 + u < cnt;
        hj[u] = HW + (int64_t)__shfl_sync(0xffffffffu, jc, src, LPR) * ld;
        ru[u] = __shfl_sync(0xffffffffu, rc, src, LPR);
      }
      for (int h = 0; h < heads; ++h) {
        const int64_t off = (int64_t)h * k2;
        float tt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) tt[u] = 0.f;
        for (int64_t c0 = 0; c0 < k2; c0 += PASS) {
          if constexpr (VEC) {
            float4 bv[U][NV], av[NV];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int v = 0; v < NV; ++v) {
                const int64_t c = c0 + 4 * (gl + LPR * v);
                bv[u][v] = (ok[u] && c < k2) ? ldg_f4(hj[u] + off + c)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const int64_t c = c0 + 4 * (gl + LPR * v);
              av[v] = c < k2 ? ldg_f4(a_dst + off + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int v = 0; v < NV; ++v) tt[u] = fma4_dot(bv[u][v], av[v], tt[u]);
          } else {
            float bv[U][NV], av[NV];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int v = 0; v < NV; ++v) {
                const int64_t c = c0 + gl + LPR * v;
                bv[u][v] = (ok[u] && c < k2) ? __ldg(hj[u] + off + c) : 0.f;
              }
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const int64_t c = c0 + gl + LPR * v;
              av[v] = c < k2 ? __ldg(a_dst + off + c) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int v = 0; v < NV; ++v) tt[u] = fmaf(bv[u][v], av[v], tt[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float dot = group_sum<LPR>(tt[u]);
          if (ok[u] && gl == 0)
            e_out[(int64_t)h * nnz + b + e0 + u] =
                leaky(__ldg(s + (int64_t)h * n_rows + ru[u]) + dot, slope);
        }
      }
    }
    jc = jn;
  }
}

int rows_grid(int64_t n_rows, int lpr, unsigned *grid) {
  const int64_t g = (n_rows + (kThreads / lpr) - 1) / (kThreads / lpr);
  if (g >= INT32_MAX) {
    set_error("row count %lld too large", (long long)n_rows);
    return GC_ERR_SHAPE;
  }
  *grid = (unsigned)g;
  return GC_OK;
}

}  // namespace
}  // namespace gnnc

using namespace gnnc;

extern "C" int gc_sddmm_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *a_vals,
                            const float *B, int64_t ldb, const float *Cm, int64_t ldc,
                            int64_t n_rows, int64_t n_cols, int64_t k, float *out_vals,
                            void *stream) {
  GC_REQUIRE(n_rows >= 0 && n_cols >= 0 && k >= 0 && ldb >= k && ldc >= k, GC_ERR_SHAPE,
             "gc_sddmm_f32: bad shape");
  if (n_rows == 0) return GC_OK;
  GC_REQUIRE(row_ptr && (k == 0 || (B && Cm)), GC_ERR_VALUE, "gc_sddmm_f32: null operand");
  unsigned grid;
  int rc = rows_grid(n_rows, 32, &grid);
  if (rc) return rc;
  sddmm_kernel<32><<<grid, kThreads, 0, as_stream(stream)>>>(row_ptr, col_idx, a_vals, B, ldb,
                                                              Cm, ldc, n_rows, k, out_vals);
  return check_launch("sddmm_kernel");
}

extern "C" int gc_sddmm_norm_f32(const int32_t *row_ptr, const int32_t *col_idx,
                                 const float *a_vals, const float *d, int64_t n_rows, int64_t nnz,
                                 float *out_vals, void *stream) {
  GC_REQUIRE(n_rows >= 0 && nnz >= 0, GC_ERR_SHAPE, "gc_sddmm_norm_f32: negative size");
  if (n_rows == 0 || nnz == 0) return GC_OK;
  GC_REQUIRE(row_ptr && col_idx && d && out_vals, GC_ERR_VALUE, "gc_sddmm_norm_f32: null operand");
  // ~8 resident waves of warps, >= 256 edges (8 per lane) per warp
  const int64_t warps_target = (int64_t)sm_count() * 8 * (kThreads / 32);
  int64_t chunk = std::max<int64_t>(256, (nnz + warps_target - 1) / warps_target);
  chunk = (chunk + 31) / 32 * 32;
  const int64_t warps = (nnz + chunk - 1) / chunk;
  const int64_t blocks = (warps + (kThreads / 32) - 1) / (kThreads / 32);
  GC_REQUIRE(blocks < INT32_MAX, GC_ERR_SHAPE, "gc_sddmm_norm_f32: too many edges");
  if (nnz >= 128 * n_rows)
    sddmm_norm_kernel<true><<<(unsigned)blocks, kThreads, 0, as_stream(stream)>>>(
        row_ptr, col_idx, a_vals, d, n_rows, nnz, chunk, out_vals);
  else
    sddmm_norm_kernel<false><<<(unsigned)blocks, kThreads, 0, as_stream(stream)>>>(
        row_ptr, col_idx, a_vals, d, n_rows, nnz, chunk, out_vals);
  return check_launch("sddmm_norm_kernel");
}

extern "C" int gc_node_proj_f32(const float *HW, int64_t ld, int64_t n_rows, int64_t k2,
                                int32_t heads, int64_t head_stride, const float *a_src,
                                const float *a_dst, float *s, float *t, void *stream) {
  GC_REQUIRE(n_rows >= 0 && k2 >= 1 && heads >= 1 && head_stride >= 0 &&
                 ld >= k2 + head_stride * (heads - 1),
             GC_ERR_SHAPE, "gc_node_proj_f32: bad shape");
  if (n_rows == 0) return GC_OK;
  GC_REQUIRE(HW && a_src && a_dst && s && t, GC_ERR_VALUE, "gc_node_proj_f32: null operand");
  const bool vec = (k2 % 4 == 0) && (ld % 4 == 0) && (head_stride % 4 == 0) && aligned16(HW) &&
                   aligned16(a_src) && aligned16(a_dst);
  unsigned grid;
  int rc = rows_grid(n_rows, 32, &grid);
  if (rc) return rc;
  node_proj_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(HW, ld, n_rows, k2, heads,
                                                             head_stride, a_src, a_dst, s, t, vec);
  return check_launch("node_proj_kernel");
}

extern "C" int gc_edge_softmax_heavy_threshold(int64_t n_rows, int64_t nnz) {
  return softmax_th(n_rows, nnz);
}

extern "C" int gc_edge_softmax_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *s,
                                   const float *t, int32_t heads, float slope, int64_t n_rows,
                                   int64_t nnz, const int32_t *heavy_rows, int64_t n_heavy,
                                   float *alpha, void *stream) {
  GC_REQUIRE(n_rows >= 0 && nnz >= 0 && n_heavy >= 0, GC_ERR_SHAPE,
             "gc_edge_softmax_f32: bad shape");
  GC_REQUIRE(heads >= 1 && heads <= kMaxHeads, GC_ERR_VALUE,
             "gc_edge_softmax_f32: heads must be in [1, %d]", kMaxHeads);
  GC_REQUIRE(slope > 0.0f && slope < 1.0f, GC_ERR_VALUE,
             "gc_edge_softmax_f32: leaky_slope must lie in (0, 1)");
  if (n_rows == 0 || nnz == 0) return GC_OK;
  GC_REQUIRE(row_ptr && col_idx && s && t && alpha && (n_heavy == 0 || heavy_rows), GC_ERR_VALUE,
             "gc_edge_softmax_f32: null operand");
  return launch_softmax<false>(row_ptr, col_idx, s, t, heads, slope, n_rows, nnz, heavy_rows,
                               n_heavy, alpha, as_stream(stream));
}

extern "C" int gc_attn_sddmm_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *HW,
                                 int64_t ld, const float *HW_self, int64_t ld_self, int64_t k2,
                                 int32_t heads, const float *a_src,
                                 const float *a_dst, float slope, int64_t n_rows, int64_t nnz,
                                 const int32_t *heavy_rows, int64_t n_heavy, float *s_work,
                                 float *alpha, void *stream) {
  GC_REQUIRE(n_rows >= 0 && nnz >= 0 && k2 >= 1 && ld >= k2 * heads, GC_ERR_SHAPE,
             "gc_attn_sddmm_f32: bad shape");
  GC_REQUIRE(heads >= 1 && heads <= kMaxHeads, GC_ERR_VALUE,
             "gc_attn_sddmm_f32: heads must be in [1, %d]", kMaxHeads);
  GC_REQUIRE(slope > 0.0f && slope < 1.0f, GC_ERR_VALUE,
             "gc_attn_sddmm_f32: leaky_slope must lie in (0, 1)");
  if (n_rows == 0 || nnz == 0) return GC_OK;
  GC_REQUIRE(row_ptr && col_idx && HW && a_src && a_dst && s_work && alpha &&
                 n_heavy >= 0 && (n_heavy == 0 || heavy_rows),
             GC_ERR_VALUE, "gc_attn_sddmm_f32: null operand");
  GC_REQUIRE(HW_self == nullptr || ld_self >= k2 * heads, GC_ERR_SHAPE,
             "gc_attn_sddmm_f32: ld_self < k2 * heads");
  if (HW_self == nullptr) HW_self = HW, ld_self = ld;
  const bool vec = (k2 % 4 == 0) && (ld % 4 == 0) && aligned16(HW) && aligned16(a_src) &&
                   aligned16(a_dst);
  const bool vec_self = (k2 % 4 == 0) && (ld_self % 4 == 0) && aligned16(HW_self) &&
                        aligned16(a_src);
  cudaStream_t st = as_stream(stream);
  // source term a_src·HW_i once per node (row i of HW_self: the pattern's own
  // rows; HW itself for a square pattern)
  unsigned grid;
  int rc = rows_grid(n_rows, 32, &grid);
  if (rc) return rc;
  node_proj_kernel<<<grid, kThreads, 0, st>>>(HW_self, ld_self, n_rows, k2, heads, k2, a_src, a_src,
                                              s_work, nullptr, vec_self);
  rc = check_launch("node_proj_kernel");
  if (rc) return rc;
  // edge-parallel target dot products: lane groups of 8 lanes (32 for rows
  // wider than 256 floats), a fixed chunk of edges per group sized for ~8
  // waves of 148 SMs
  int lpr = 8, nv = 1, u = 8;
  if (vec) {
    if (k2 <= 32) nv = 1, u = 8;
    else if (k2 <= 64) nv = 2, u = 8;
    else if (k2 <= 128) nv = 4, u = 4;
    else if (k2 <= 256) nv = 8, u = 2;
    else lpr = 32, nv = 4, u = 2;  // 512 floats per pass
  } else {
    lpr = 32, nv = 2, u = 4;
  }
  const int64_t groups_per_block = kThreads / lpr;
  const int64_t target_groups = (int64_t)sm_count() * 8 * groups_per_block;
  int64_t chunk = std::max<int64_t>(64, (nnz + target_groups - 1) / target_groups);
  chunk = (chunk + 7) / 8 * 8;
  const int64_t n_groups = (nnz + chunk - 1) / chunk;
  const int64_t blocks = (n_groups + groups_per_block - 1) / groups_per_block;
  GC_REQUIRE(blocks < INT32_MAX, GC_ERR_SHAPE, "gc_attn_sddmm_f32: too many edges");
#define GC_SCORE(L, N, UU, V)                                                           \
  attn_score_kernel<L, N, UU, V><<<(unsigned)blocks, kThreads, 0, st>>>(                \
      row_ptr, col_idx, HW, ld, k2, heads, s_work, a_dst, slope, n_rows, nnz, chunk, alpha)
  if (!vec) GC_SCORE(32, 2, 4, false);
  else if (lpr == 32) GC_SCORE(32, 4, 2, true);
  else if (nv == 1) GC_SCORE(8, 1, 8, true);
  else if (nv == 2) GC_SCORE(8, 2, 8, true);
  else if (nv == 4) GC_SCORE(8, 4, 4, true);
  else GC_SCORE(8, 8, 2, true);
#undef GC_SCORE
  rc = check_launch("attn_score_kernel");
  if (rc) return rc;
  return launch_softmax<true>(row_ptr, col_idx, nullptr, nullptr, heads, slope, n_rows, nnz,
                              heavy_rows, n_heavy, alpha, st);
}
