// Edge-wise kernels over the CSR pattern: SDDMM (sparse.py:222-232), the k=1
// normalisation SDDMM (gcn.py:103-112) and the GAT attention in both
// compositions (gat.py:72-114): the reassociated per-node projections + fused
// LeakyReLU/edge-softmax, and the SDDMM-over-edges variant.
//
// All of these are HBM-bound streams over col_idx (+ values) with an L2-resident
// per-node gather (d, t); each row is owned by one lane group, the reductions
// use a fixed shuffle tree, so results are deterministic.
#include <math.h>

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

// k = 1 normalisation: out[p] = a[p] * (d[i] * d[j])
template <int LPR>
__global__ void __launch_bounds__(kThreads)
    sddmm_norm_kernel(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                      const float *__restrict__ a_vals, const float *__restrict__ d,
                      int64_t n_rows, float *__restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * (kThreads / LPR) + threadIdx.x / LPR;
  const int gl = threadIdx.x % LPR;
  if (row >= n_rows) return;
  const int beg = row_ptr[row], end = row_ptr[row + 1];
  const float di = __ldg(d + row);
  for (int p = beg + gl; p < end; p += LPR) {
    const float prod = di * __ldg(d + ldg_stream_i32(col_idx + p));
    out[p] = (a_vals ? ldg_stream_f32(a_vals + p) : 1.0f) * prod;
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
      t[(int64_t)h * n_rows + row] = tt;
    }
  }
}

// ---------------------------------------------------------------------------
// fused LeakyReLU + edge softmax (reassociated attention), multi-head.
// Pass 1: per-lane online (max, sum); group merge.  Pass 2: normalised write.
// ---------------------------------------------------------------------------
template <int LPR>
__global__ void __launch_bounds__(kThreads)
    edge_softmax_kernel(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                        const float *__restrict__ s, const float *__restrict__ t, int heads,
                        float slope, int64_t n_rows, int64_t nnz, float *__restrict__ alpha) {
  const int64_t row = (int64_t)blockIdx.x * (kThreads / LPR) + threadIdx.x / LPR;
  const int gl = threadIdx.x % LPR;
  const bool live = row < n_rows;
  const int beg = live ? row_ptr[row] : 0, end = live ? row_ptr[row + 1] : 0;
  float si[kMaxHeads], m[kMaxHeads], z[kMaxHeads];
#pragma unroll
  for (int h = 0; h < kMaxHeads; ++h) {
    si[h] = (live && h < heads) ? __ldg(s + (int64_t)h * n_rows + row) : 0.f;
    m[h] = -INFINITY;
    z[h] = 0.f;
  }
  for (int p = beg + gl; p < end; p += LPR) {
    const int j = __ldg(col_idx + p);
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
      if (h >= heads) break;
      const float e = leaky(si[h] + __ldg(t + (int64_t)h * n_rows + j), slope);
      if (e > m[h]) {
        z[h] = z[h] * expf(m[h] - e) + 1.0f;
        m[h] = e;
      } else {
        z[h] += expf(e - m[h]);
      }
    }
  }
#pragma unroll
  for (int h = 0; h < kMaxHeads; ++h) {
    if (h >= heads) break;
    const float mg = group_max<LPR>(m[h]);
    const float zl = (m[h] == -INFINITY) ? 0.f : z[h] * expf(m[h] - mg);
    z[h] = group_sum<LPR>(zl);
    m[h] = mg;
  }
  if (!live || end == beg) return;
  for (int p = beg + gl; p < end; p += LPR) {
    const int j = __ldg(col_idx + p);
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
      if (h >= heads) break;
      const float e = leaky(si[h] + __ldg(t + (int64_t)h * n_rows + j), slope);
      alpha[(int64_t)h * nnz + p] = expf(e - m[h]) / z[h];
    }
  }
}

// ---------------------------------------------------------------------------
// attention as an SDDMM over edges: e = a_src·HW_i + a_dst·HW_j per edge
// (k2-wide dot products, warp per row, lanes across the k2 columns), then
// the same LeakyReLU + softmax.  Raw scores are staged in `alpha`.
// ---------------------------------------------------------------------------
template <bool VEC>
__global__ void __launch_bounds__(kThreads)
    attn_sddmm_kernel(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                      const float *__restrict__ HW, int64_t ld, int64_t k2, int heads,
                      const float *__restrict__ a_src, const float *__restrict__ a_dst,
                      float slope, int64_t n_rows, int64_t nnz, float *__restrict__ alpha) {
  const int64_t row = (int64_t)blockIdx.x * (kThreads / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= n_rows) return;
  const int beg = row_ptr[row], end = row_ptr[row + 1];
  if (beg == end) return;
  const float *hi = HW + row * ld;
  for (int h = 0; h < heads; ++h) {
    const int64_t off = (int64_t)h * k2;
    const float *al = a_src + off;
    const float *ar = a_dst + off;
    // per-row source term
    float ss = 0.f;
    if (VEC) {
      for (int64_t c = 4 * lane; c < k2; c += 128) ss = fma4_dot(ldg_f4(hi + off + c), ldg_f4(al + c), ss);
    } else {
      for (int64_t c = lane; c < k2; c += 32) ss = fmaf(__ldg(hi + off + c), __ldg(al + c), ss);
    }
    ss = group_sum<32>(ss);
    float m = -INFINITY, z = 0.f;
    float *ah = alpha + (int64_t)h * nnz;
    int p = beg;
    // 4 edges per step keeps 4 independent row gathers in flight per lane
    for (; p + 4 <= end; p += 4) {
      float tt[4] = {0.f, 0.f, 0.f, 0.f};
      const float *hj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) hj[u] = HW + (int64_t)__ldg(col_idx + p + u) * ld + off;
      if (VEC) {
        for (int64_t c = 4 * lane; c < k2; c += 128) {
          const float4 a = ldg_f4(ar + c);
#pragma unroll
          for (int u = 0; u < 4; ++u) tt[u] = fma4_dot(ldg_f4(hj[u] + c), a, tt[u]);
        }
      } else {
        for (int64_t c = lane; c < k2; c += 32) {
          const float a = __ldg(ar + c);
#pragma unroll
          for (int u = 0; u < 4; ++u) tt[u] = fmaf(__ldg(hj[u] + c), a, tt[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float e = leaky(ss + group_sum<32>(tt[u]), slope);
        if (lane == u) ah[p + u] = e;
        const float mn = fmaxf(m, e);
        z = z * expf(m - mn) + expf(e - mn);
        m = mn;
      }
    }
    for (; p < end; ++p) {
      const float *hj = HW + (int64_t)__ldg(col_idx + p) * ld + off;
      float tt = 0.f;
      if (VEC) {
        for (int64_t c = 4 * lane; c < k2; c += 128) tt = fma4_dot(ldg_f4(hj + c), ldg_f4(ar + c), tt);
      } else {
        for (int64_t c = lane; c < k2; c += 32) tt = fmaf(__ldg(hj + c), __ldg(ar + c), tt);
      }
      const float e = leaky(ss + group_sum<32>(tt), slope);
      if (lane == 0) ah[p] = e;
      const float mn = fmaxf(m, e);
      z = z * expf(m - mn) + expf(e - mn);
      m = mn;
    }
    __syncwarp();
    for (int q = beg + lane; q < end; q += 32) ah[q] = expf(ah[q] - m) / z;
    __syncwarp();
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
  if (n_rows == 0) return GC_OK;
  GC_REQUIRE(row_ptr && d, GC_ERR_VALUE, "gc_sddmm_norm_f32: null operand");
  // lanes per row follow the mean degree: short rows share a warp, long rows
  // get the whole warp (the per-edge d_j gather is latency-bound otherwise)
  const bool wide = nnz > 12 * n_rows;
  unsigned grid;
  cudaStream_t st = as_stream(stream);
  int rc = rows_grid(n_rows, wide ? 32 : 8, &grid);
  if (rc) return rc;
  if (wide)
    sddmm_norm_kernel<32><<<grid, kThreads, 0, st>>>(row_ptr, col_idx, a_vals, d, n_rows, out_vals);
  else
    sddmm_norm_kernel<8><<<grid, kThreads, 0, st>>>(row_ptr, col_idx, a_vals, d, n_rows, out_vals);
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

extern "C" int gc_edge_softmax_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *s,
                                   const float *t, int32_t heads, float slope, int64_t n_rows,
                                   int64_t nnz, float *alpha, void *stream) {
  GC_REQUIRE(n_rows >= 0 && nnz >= 0, GC_ERR_SHAPE, "gc_edge_softmax_f32: bad shape");
  GC_REQUIRE(heads >= 1 && heads <= kMaxHeads, GC_ERR_VALUE,
             "gc_edge_softmax_f32: heads must be in [1, %d]", kMaxHeads);
  GC_REQUIRE(slope > 0.0f && slope < 1.0f, GC_ERR_VALUE,
             "gc_edge_softmax_f32: leaky_slope must lie in (0, 1)");
  if (n_rows == 0 || nnz == 0) return GC_OK;
  GC_REQUIRE(row_ptr && col_idx && s && t && alpha, GC_ERR_VALUE,
             "gc_edge_softmax_f32: null operand");
  cudaStream_t st = as_stream(stream);
  unsigned grid;
  const double avg = (double)nnz / (double)n_rows;
  if (avg <= 12.0) {
    int rc = rows_grid(n_rows, 8, &grid);
    if (rc) return rc;
    edge_softmax_kernel<8><<<grid, kThreads, 0, st>>>(row_ptr, col_idx, s, t, heads, slope,
                                                      n_rows, nnz, alpha);
  } else {
    int rc = rows_grid(n_rows, 32, &grid);
    if (rc) return rc;
    edge_softmax_kernel<32><<<grid, kThreads, 0, st>>>(row_ptr, col_idx, s, t, heads, slope,
                                                       n_rows, nnz, alpha);
  }
  return check_launch("edge_softmax_kernel");
}

extern "C" int gc_attn_sddmm_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *HW,
                                 int64_t ld, int64_t k2, int32_t heads, const float *a_src,
                                 const float *a_dst, float slope, int64_t n_rows, int64_t nnz,
                                 float *alpha, void *stream) {
  GC_REQUIRE(n_rows >= 0 && nnz >= 0 && k2 >= 1 && ld >= k2 * heads, GC_ERR_SHAPE,
             "gc_attn_sddmm_f32: bad shape");
  GC_REQUIRE(heads >= 1 && heads <= kMaxHeads, GC_ERR_VALUE,
             "gc_attn_sddmm_f32: heads must be in [1, %d]", kMaxHeads);
  GC_REQUIRE(slope > 0.0f && slope < 1.0f, GC_ERR_VALUE,
             "gc_attn_sddmm_f32: leaky_slope must lie in (0, 1)");
  if (n_rows == 0 || nnz == 0) return GC_OK;
  GC_REQUIRE(row_ptr && col_idx && HW && a_src && a_dst && alpha, GC_ERR_VALUE,
             "gc_attn_sddmm_f32: null operand");
  unsigned grid;
  int rc = rows_grid(n_rows, 32, &grid);
  if (rc) return rc;
  const bool vec = (k2 % 4 == 0) && (ld % 4 == 0) && aligned16(HW) && aligned16(a_src) &&
                   aligned16(a_dst);
  cudaStream_t st = as_stream(stream);
  if (vec)
    attn_sddmm_kernel<true><<<grid, kThreads, 0, st>>>(row_ptr, col_idx, HW, ld, k2, heads, a_src,
                                                       a_dst, slope, n_rows, nnz, alpha);
  else
    attn_sddmm_kernel<false><<<grid, kThreads, 0, st>>>(row_ptr, col_idx, HW, ld, k2, heads,
                                                        a_src, a_dst, slope, n_rows, nnz, alpha);
  return check_launch("attn_sddmm_kernel");
}
