// Dense update H·W for sm_100a (replaces gnncompose/sparse.py:285-291, gemm).
//
// Two kernels behind gc_gemm_f32:
//  * gemm_tf32_tcgen05: TMA (SWIZZLE_128B) -> smem ring -> tcgen05.mma
//    kind::tf32 (one elected thread issues) -> fp32 accumulators in TMEM ->
//    tcgen05.ld epilogue with the row scale (D^-1/2) and ReLU fused.
//    Both operands are K-major: A = H (row-major M x K) as is, B = W^T, which
//    a tiny transpose kernel writes into the caller's workspace.
//  * gemm_fp32_simt: exact-fp32 CUDA-core tiles; the rtol-1e-4 parity mode and
//    the path for operands TMA cannot describe (lda % 4 != 0, e.g. Cora's
//    k1 = 1433).
// Plus gc_scale_rows_f32 (D^-1/2 X / ReLU as a standalone pass).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace gnnc {
namespace {

// ============================================================================
// small PTX wrappers (tcgen05 / TMA / mbarrier)
// ============================================================================
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint64_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++spins > (1ull << 26)) __trap();
  }
}

// The same with cluster-scope acquire: the waiter then observes the
// (release.cluster) arrivals' prior shared-memory writes of the peer CTA.
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint64_t spins = 0;
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    if (++spins > (1ull << 26)) __trap();
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

// plain bulk copy global -> this CTA's shared memory (16-B aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_load_1d(uint32_t dst, const void *src, uint32_t bytes,
                                             uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t src, int32_t c0,
                                             int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// one lane of a converged warp (the same lane every call)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major operand in a 128-byte-swizzled tile: rows of 128 B, 8-row atoms of
// 1024 B stacked along M/N (SBO = 1024 B), LBO unused (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;             // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

// MN-major SWIZZLE_128B operand (16-bit): 64-element MN rows of 128 B, 8-row
// (K) atoms of 1 KB at SBO = 1 KB, MN blocks of 64 elements at LBO = lbo bytes
// (the layout a 2-D TMA box {64 MN, rows K} with SWIZZLE_128B writes).
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor: D = F32, A = B = TF32, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

// Instruction descriptor: D = F32, A = B = BF16 (kind::f16), both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
// D = F32, A = B = F16 (kind::f16, format 0), both K-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ============================================================================
// tcgen05 TF32 GEMM
// ============================================================================
constexpr int BM = 128;             // UMMA_M (cta_group::1)
constexpr int BK = 32;              // fp32 elements per 128-byte swizzle row
constexpr int UMMA_K = 8;           // K per tcgen05.mma for kind::tf32
// Both element types use the same byte geometry: a k-block is one 128-byte
// swizzle row (32 fp32 or 64 bf16) and one MMA consumes 32 bytes of it
// (8 tf32 or 16 bf16), so the descriptors, TMA boxes and ring are shared.
constexpr int KB_BYTES = 128;
constexpr int MMA_K_BYTES = 32;
// 6 warps: 0 = TMA producer (+ TMEM alloc), 1 = MMA issuer, 2..5 = epilogue.
// Epilogue warp w reads TMEM lanes 32*(w%4) .. +31, so warps 2..5 cover all 128.
constexpr int kGemmThreads = 192;

struct GemmEpi {
  float *C;
  int64_t ldc;
  const float *row_scale;
  int64_t M, N;
  uint32_t flags;
  const float *scale;  // optional device scalar multiplied into every row (f16x2 unscale)
  // fp16-row output (gc_gemm_f16rows_f32, the TF32 class's gather operand):
  // Ch[row, chunk] = fp16_rn(out * 2^-e), sigma[row * sig_ld + chunk] = 2^e,
  // each N tile's row max in [2^14, 2^15) — one scale per row when the row
  // is one tile (BN >= N), one per 256-column chunk otherwise (sig_ld chunks)
  __half *Ch;
  int64_t ldh;
  float *sigma;
  int sig_ld;
};

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Persistent warp-specialised TF32 GEMM.  Tiles (BM x BN) are walked
// n-fastest (consecutive tiles of a CTA reuse the same A rows from L2); the
// smem ring streams k-blocks across tile boundaries, and the accumulator is
// double-buffered in TMEM (2 x BN columns) so the epilogue of tile i overlaps
// the mainloop of tile i+1.
//
// TERMS > 1 (the dense hub block of the hybrid aggregation, BF16): the B
// operand is TERMS stacked [b_rows_per_term x K] slices (hi/mid/lo bf16 terms
// of one fp32 operand); each k-block stages one A tile and TERMS B tiles and
// issues TERMS MMAs per 32-byte step into the same accumulator, so
// D = A·(B0 + B1 + B2) with the A tile read once.
// ELEM: 0 = TF32 (kind::tf32), 1 = BF16, 2 = FP16 (kind::f16)
//
// SPLITA (TF32 only, TERMS = 2: B = [hi(W^T); lo(W^T)]): the 3xTF32
// fp32-class product.  Four converter warps (6..9) rewrite each landed A tile
// in place as hi = A with the 13 low mantissa bits cleared (exact in TF32)
// and write lo = A - hi (exact in fp32) to a second tile of the stage; the
// MMA warp then issues hi·hi + hi·lo + lo·hi per 32-byte step.  The dropped
// lo·lo term and the TF32 rounding of lo are both ~2^-20 of |a·b|, so the
// result carries ~fp32 accuracy (normwise ~1e-6) at three TF32 MMAs.
constexpr int kConvThreads = 128;
template <int BN, int TERMS, int ELEM, bool SPLITA = false>
__device__ __forceinline__ void gemm_tc_body(const CUtensorMap &map_a, const CUtensorMap &map_b,
                                             const CUtensorMap &map_c, const GemmEpi &ep,
                                             int num_kb, int stages, int m_tiles, int n_tiles,
                                             int tma_store, int b_rows_per_term) {
  static_assert(!SPLITA || (ELEM == 0 && TERMS == 2), "3xTF32 split: TF32 with B = [hi; lo]");
  constexpr uint32_t A_BYTES = BM * KB_BYTES;
  constexpr uint32_t ALO_BYTES = SPLITA ? A_BYTES : 0u;  // lo(A) tile written by the converters
  constexpr uint32_t B_BYTES = BN * KB_BYTES;
  constexpr uint32_t B_OFF = A_BYTES + ALO_BYTES;
  constexpr uint32_t STAGE_BYTES = B_OFF + TERMS * B_BYTES;
  constexpr bool BF16 = ELEM != 0;  // 16-bit elements (kind::f16)
  constexpr int KB_ELEMS = BF16 ? 64 : 32;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // power of two >= 32

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SWIZZLE_128B needs 1024-B alignment
  uint8_t *gbase = smem_raw + (base - raw);
  const uint32_t bar0 = base + (uint32_t)stages * STAGE_BYTES;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (stages + s); };
  auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * stages + b); };
  auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * stages + 2 + b); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + (bar0 - base) + 8u * (2 * stages + 4));
  // SPLITA: per-stage "A converted" barriers after the TMEM slot
  auto conv_bar = [&](int s) { return bar0 + 8u * (2 * stages + 4) + 16u + 8u * s; };
  // epilogue staging: per epilogue warp 2 x (32 rows x 16 fp32) boxes, 64-B swizzled
  const uint32_t stage_c =
      (bar0 + 8u * (2 * stages + 4) + 16u + (SPLITA ? 8u * stages : 0u) + 1023u) & ~1023u;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_tiles_total = m_tiles * n_tiles;

  if (warp == 1 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int s = 0; s < stages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 4);  // one arrive per epilogue warp
    }
    if constexpr (SPLITA)
      for (int s = 0; s < stages; ++s) mbar_init(conv_bar(s), kConvThreads / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x) {
        const int m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(empty_bar(s), ((it / stages) & 1) ^ 1);
          const uint32_t sa = base + (uint32_t)s * STAGE_BYTES;
          mbar_expect_tx(full_bar(s), STAGE_BYTES - ALO_BYTES);  // TMA bytes (lo(A) is made on chip)
          tma_load_2d(sa, &map_a, full_bar(s), kb * KB_ELEMS, m0);
#pragma unroll
          for (int q = 0; q < TERMS; ++q)
            tma_load_2d(sa + B_OFF + q * B_BYTES, &map_b, full_bar(s), kb * KB_ELEMS,
                        q * b_rows_per_term + n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer (one thread) ----------------
      constexpr uint32_t idesc = ELEM == 2 ? idesc_f16(BN) : ELEM == 1 ? idesc_bf16(BN) : idesc_tf32(BN);
      int it = 0, lt = 0;
      for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x, ++lt) {
        const int acc = lt & 1;
        mbar_wait(tempty_bar(acc), ((lt >> 1) & 1) ^ 1);  // epilogue drained this buffer
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % stages;
          // SPLITA: the converters' arrival implies the TMA bytes landed
          mbar_wait(SPLITA ? conv_bar(s) : full_bar(s), (it / stages) & 1);
          tc_fence_after();
          const uint32_t sa = base + (uint32_t)s * STAGE_BYTES;
#pragma unroll
          for (int k = 0; k < KB_BYTES / MMA_K_BYTES; ++k) {
            const uint64_t ad = umma_desc_sw128(sa + k * MMA_K_BYTES);
            if constexpr (SPLITA) {
              const uint64_t alo = umma_desc_sw128(sa + A_BYTES + k * MMA_K_BYTES);
              const uint64_t bhi = umma_desc_sw128(sa + B_OFF + k * MMA_K_BYTES);
              const uint64_t blo = umma_desc_sw128(sa + B_OFF + B_BYTES + k * MMA_K_BYTES);
              mma_tf32(tmem_d, alo, bhi, idesc, (kb | k) != 0);  // small terms first
              mma_tf32(tmem_d, ad, blo, idesc, 1);
              mma_tf32(tmem_d, ad, bhi, idesc, 1);
              continue;
            }
#pragma unroll
            for (int q = 0; q < TERMS; ++q) {
              const uint64_t bd = umma_desc_sw128(sa + B_OFF + q * B_BYTES + k * MMA_K_BYTES);
              if constexpr (BF16) mma_bf16(tmem_d, ad, bd, idesc, (kb | k | q) != 0);
              else mma_tf32(tmem_d, ad, bd, idesc, (kb | k | q) != 0);
            }
          }
          mma_commit(empty_bar(s));  // frees the smem slot once these MMAs retire
        }
        mma_commit(tfull_bar(acc));  // accumulator of this tile complete
      }
    }
  } else if (SPLITA && warp >= kGemmThreads / 32) {  // -------- A-split converters --------
    // thread t rewrites 16-byte chunks t, t+128, ... of the landed A tile:
    // each warp access is 512 contiguous bytes (conflict-free); the swizzle
    // is irrelevant to an elementwise map as hi / lo keep A's positions
    const int ct = threadIdx.x - kGemmThreads;
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x) {
      for (int kb = 0; kb < num_kb; ++kb, ++it) {
        const int s = it % stages;
        mbar_wait(full_bar(s), (it / stages) & 1);
        uint8_t *ta = gbase + (size_t)s * STAGE_BYTES;
#pragma unroll
        for (int i = 0; i < (int)(A_BYTES / 16 / kConvThreads); ++i) {
          const uint32_t off = (uint32_t)(i * kConvThreads + ct) * 16u;
          float4 *pa = reinterpret_cast<float4 *>(ta + off);
          const float4 v = *pa;
          float4 hi;
          hi.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          hi.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          hi.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          hi.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          *pa = hi;
          *reinterpret_cast<float4 *>(ta + A_BYTES + off) =
              make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
        }
        fence_proxy_async_smem();  // generic-proxy stores -> visible to the MMA (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(conv_bar(s));
      }
    }
  } else {  // ---------------- epilogue warps 2..5 ----------------
    // TMEM -> registers (thread = row, 16 consecutive columns per tcgen05.ld)
    // -> fused row scale / ReLU -> 4 x 16-byte stores per row segment.  (A
    // shared-memory transpose for line-coalesced stores measured slower: it
    // triples the epilogue's instruction count; profiles/r01_ncu_summary.md.)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const bool relu = (ep.flags & GC_RELU) != 0;
    const bool accum = (ep.flags & GC_ACCUMULATE) != 0;
    const bool vec = ((ep.ldc & 3) == 0) && aligned16(ep.C);
    const uint32_t my_stage = stage_c + (uint32_t)(warp - 2) * 2u * 2048u;
    int lt = 0, sbuf = 0;
    for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      const int m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
      mbar_wait(tfull_bar(acc), (lt >> 1) & 1);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < ep.M;
      float rs = (row_ok && ep.row_scale) ? __ldg(ep.row_scale + row) : 1.0f;
      if (ep.scale) rs *= __ldg(ep.scale);
      float *crow = ep.C + (int64_t)row * ep.ldc;
      const uint32_t taddr = tmem_base + (uint32_t)(acc * BN) + ((uint32_t)(q * 32) << 16);
      if (ep.Ch) {
        // fp16 rows (TF32 class): pass 1 finds the tile row's max in TMEM,
        // pass 2 converts with the exact power-of-two scale (one scale per
        // row and N tile: the whole row when BN >= N, else 256-column chunks)
        const int nv = ep.N - n0;  // valid columns of this tile
        float mx = 0.0f;
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          if (c >= nv) break;  // warp-uniform
          float v[16];
          tmem_ld16(taddr + (uint32_t)c, v);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c + i < nv) mx = fmaxf(mx, fabsf(v[i] * rs));
        }
        const int E = mx > 0.0f ? ((int)((__float_as_uint(mx) >> 23) & 0xff) - 127) : 0;
        const int e = mx > 0.0f && isfinite(mx) ? max(min(E - 14, 110), -110) : 0;
        const float down = __uint_as_float((uint32_t)(127 - e) << 23) * rs;
        __half *hrow = ep.Ch + (int64_t)row * ep.ldh + n0;
        const int64_t nh = ep.ldh - n0;  // padded columns of this tile
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          if (c >= nh) break;  // warp-uniform (ldh: N rounded up to 8)
          float v[16];
          tmem_ld16(taddr + (uint32_t)c, v);
          if (!row_ok) continue;
          __half2 hv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            hv[i] = __floats2half2_rn(c + 2 * i < nv ? v[2 * i] * down : 0.0f,
                                      c + 2 * i + 1 < nv ? v[2 * i + 1] * down : 0.0f);
          if (c + 16 <= nh) {
            uint4 *dst = reinterpret_cast<uint4 *>(hrow + c);
            dst[0] = *reinterpret_cast<const uint4 *>(&hv[0]);
            dst[1] = *reinterpret_cast<const uint4 *>(&hv[4]);
          } else {  // the last 8 halves of a row whose padded width is 8 mod 16
            *reinterpret_cast<uint4 *>(hrow + c) = *reinterpret_cast<const uint4 *>(&hv[0]);
          }
        }
        if (row_ok)
          ep.sigma[(int64_t)row * ep.sig_ld + n0 / BN] = __uint_as_float((uint32_t)(127 + e) << 23);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty_bar(acc));
        continue;
      }
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        if (n0 + c >= ep.N) break;  // warp-uniform
        float v[16];
        tmem_ld16(taddr + (uint32_t)c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] *= rs;
          if (relu && !accum) v[i] = fmaxf(v[i], 0.0f);
        }
        if (tma_store) {  // (never with GC_ACCUMULATE: the host forces direct stores)
          // row `lane` of a 32 x 16 box: four 16-B chunks, 64-B swizzle
          // (chunk ^ ((row >> 1) & 3)) -> conflict-free st.shared.v4
          const uint32_t buf = my_stage + (uint32_t)sbuf * 2048u;
          if (lane == 0) bulk_wait_read<1>();  // this buffer's previous store has been read
          __syncwarp();
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const uint32_t dst = buf + (uint32_t)lane * 64u + (uint32_t)((ch ^ ((lane >> 1) & 3)) * 16);
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "f"(v[4 * ch]),
                         "f"(v[4 * ch + 1]), "f"(v[4 * ch + 2]), "f"(v[4 * ch + 3])
                         : "memory");
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&map_c, buf, n0 + c, m0 + q * 32);  // TMA clips rows >= M, cols >= N
            bulk_commit();
          }
          sbuf ^= 1;
          continue;
        }
        if (!row_ok) continue;
        const int64_t col = n0 + c;
        if (accum) {  // C = relu?(old + rs * acc), the SpMM epilogue's order
          if (vec && col + 16 <= ep.N) {  // 16-byte read-modify-write
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              float4 o = *reinterpret_cast<const float4 *>(crow + col + i);
              o.x += v[i], o.y += v[i + 1], o.z += v[i + 2], o.w += v[i + 3];
              if (relu) o.x = fmaxf(o.x, 0.f), o.y = fmaxf(o.y, 0.f), o.z = fmaxf(o.z, 0.f), o.w = fmaxf(o.w, 0.f);
              stg_f4(crow + col + i, o);
            }
            continue;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (col + i < ep.N) {
              float o = crow[col + i] + v[i];
              if (relu) o = fmaxf(o, 0.0f);
              crow[col + i] = o;
            }
          continue;
        }
        if (vec && col + 16 <= ep.N) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            stg_f4(crow + col + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (col + i < ep.N) crow[col + i] = v[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty_bar(acc));
    }
    if (tma_store && lane == 0) bulk_wait_all();  // stores complete before the CTA exits
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
}

// ============================================================================
// CTA-pair (cta_group::2) variant of the hub GEMM
// ============================================================================
// Two CTAs of a cluster (one TPC) share every MMA: M = 256 (each CTA stages
// its own 128 rows of A_hub) and N = BN (each CTA stages BN/2 rows of each B
// term), so per SM the B operand traffic through shared memory and L2 is
// halved — the single-CTA kernel is shared-memory-bandwidth bound (operand
// reads of N = 128 tiles plus the TMA writes exceed 128 B/clk).  Protocol:
//  * both CTAs' TMA loads complete_tx on the LEADER's full barrier (count 2:
//    leader arrive.expect_tx(both stages' bytes) + peer remote arrive);
//  * the leader's single MMA thread issues tcgen05.mma.cta_group::2 and
//    commits with a 0b11 multicast to both CTAs' empty / tmem-full barriers;
//  * the 8 epilogue warps (4 per CTA) arrive on the leader's tmem-empty barrier.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap *map,
                                                 uint32_t leader_bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap *map,
                                                 uint32_t leader_bar, int32_t c0, int32_t c1,
                                                 int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"((uint16_t)0x3)
      : "memory");
}
// D = F32, A = B = BF16, K-major, M = 256 (cta pair), N = n
__host__ __device__ constexpr uint32_t idesc_bf16_m256(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((256u >> 4) << 24);
}
// D = F32, A = B = F16, K-major, M = 256 (cta pair), N = n
__host__ __device__ constexpr uint32_t idesc_f16_m256(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((256u >> 4) << 24);
}
// D = F32, A = B = TF32, K-major, M = 256 (cta pair), N = n
__host__ __device__ constexpr uint32_t idesc_tf32_m256(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((256u >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Staircase of dense blocks (hub.py): step s is the 0/1 block of rows
// [0, rows[s]) (rows in degree-rank order) x columns [c0[s], c0[s] + 64*nkb[s])
// (column-degree-rank order, i.e. positions in the packed B operand).  Rows
// shrink as columns grow, so the columns a rank-ordered M-tile reduces over
// are a prefix of the steps; one accumulator per tile covers all of them and
// the epilogue scatters row r to row_map[r] (nullptr: identity).  One step
// with rows = n is the plain hub block.
constexpr int kMaxSteps = 16;
struct StairMaps {
  CUtensorMap a[kMaxSteps];
};
struct StairArgs {
  int n_steps;
  int rows[kMaxSteps];
  int c0[kMaxSteps];
  int nkb[kMaxSteps];
  // bit-packed blocks (GC_HUB_A_BITS): step s's words start at bits[s],
  // word (k, r) at k * rpad(s) + r, rpad = rows rounded up to 256
  const uint64_t *bits[kMaxSteps];
  const int32_t *row_map;
  // optional static schedule (longest-processing-time first, built by the
  // caller): cluster c runs work items items[cluster_start[c] ..
  // cluster_start[c+1]); item = {tile, first k-block, end k-block (-1: all),
  // workspace slot (-1: write C)} — split-K for the longest tiles
  const int4 *items;
  const int32_t *cluster_start;
  float *ws;  // [slot][256 rank rows][BN] partial products (rows pre-scaled)
  int dbg;    // experiments only (GNNC_HUB_DBG): 1 = A once per step, 2 = B once, 4 = no MMA,
              // 8 = converters skip the expansion, 16 = no proxy fence, 32 = no bitmap loads,
              // 64 = MMA ignores aready, 128 = no A-slot release, 256 = no epilogue stores
              // (timing only)
};

__device__ __forceinline__ int stair_kblocks(const StairArgs &sa, int m0) {
  int t = 0;
  for (int s = 0; s < sa.n_steps; ++s)
    if (sa.rows[s] > m0) t += sa.nkb[s];
  return t;
}

// FMT 0: three bf16 terms (exact fp32 split); 1: two fp16 terms of s·D·X
// (22 significant bits, absolute error <= 2^-23 max|D·X|), 2/3 of the MMAs;
// 2: one fp32 operand pair on kind::tf32 (the dense update H·W on CTA pairs);
// 3: one fp16 term of s·D·X (11 significant bits: TF32's input rounding).
constexpr int fmt_terms(int fmt) { return fmt >= 2 ? 1 : fmt == 1 ? 2 : 3; }

// ABITS: the 0/1 A blocks arrive as bitmaps (1 KB per 128 x 64 k-block tile
// instead of 16 KB) and converter warps expand them into the SWIZZLE_128B
// fp16/bf16 tile the MMA reads — the dense part's DRAM traffic drops to the
// B operand (L2-resident) plus 1/16 of the A bytes.  Three rings: bitmaps
// (kBitsSlots deep, streamed by a dedicated producer warp: DRAM latency is
// hidden by 1 KB slots), converted A tiles (kAStages: produced on chip, so
// shallow) and B tiles (all remaining shared memory: the B stream from L2 is
// latency x bytes-in-flight bound).  Converter groups (4 warps = 128 rows
// each) take alternate k-blocks — one group's per-k-block latency (wait,
// expand, proxy fence, remote arrive) exceeds the MMA time of a k-block.
// Group g owns A slot g (kAStages == kConvGroups): every slot's barriers have
// one sequential waiter, so no waiter can run two phases ahead (parity
// aliasing), and the bitmap slots map to groups the same way.
// Measured on Reddit K=256 (stair:8, one fp16 term): 0.86 ms vs 0.62 ms with
// 16-bit A tiles from HBM — the per-k-block handoff chain (bitmap -> converter
// -> cluster arrive -> MMA -> commit -> converter) bounds it: more A slots do
// not help (8 per 4 groups: 0.86), fewer groups hurt (2: 1.12).  Kept as the
// GC_HUB_A_BITS option for its 16x smaller block storage.
constexpr int kConvGroups = 4;
constexpr int kAStages = kConvGroups;
constexpr int kBitsSlots = 16;
static_assert(kAStages % kConvGroups == 0 && kBitsSlots % kConvGroups == 0, "bitmap slot -> converter group must be fixed");
constexpr int kBitsThreads = 32 + 128 * kConvGroups;

template <int BN, int FMT, bool ABITS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ABITS ? kGemmThreads + kBitsThreads : kGemmThreads + 32, 1)
    gemm_hub_pair_tcgen05(const __grid_constant__ StairMaps maps,
                          const __grid_constant__ CUtensorMap map_b,
                          const __grid_constant__ CUtensorMap map_c, const GemmEpi ep,
                          const StairArgs sarg, int stages, int m_pairs, int n_tiles,
                          int tma_store, int b_rows_per_term) {
  constexpr int TERMS = fmt_terms(FMT);
  constexpr int KB_EL = FMT == 2 ? 32 : 64;  // elements per 128-byte k-block row
  constexpr int BH = BN / 2;  // B rows per CTA per term
  constexpr uint32_t A_BYTES = BM * KB_BYTES;
  constexpr uint32_t B_BYTES = BH * KB_BYTES;
  constexpr uint32_t BITS_BYTES = BM * 8u;  // 128 rows x 64 bits
  constexpr uint32_t STAGE_BYTES = A_BYTES + TERMS * B_BYTES;
  static_assert(!ABITS || FMT != 2, "bitmap A is a 16-bit operand");
  // FMT 4: one fp16 term with B MN-major ([T][Kp] rows as packed, no
  // transpose): BH/64 TMA boxes of 64 features x 64 hub rows per stage
  constexpr bool MNB = FMT == 4;
  static_assert(!MNB || BH % 64 == 0, "MN-major B needs 64-element blocks per CTA");
  // Narrow tiles (BN <= 64): the three staged term tiles are one contiguous
  // K-major [3*BH rows] operand, so ONE MMA with N = 3*BN covers all terms
  // (A is read once per k-step instead of three times) and the epilogue adds
  // the three term column groups.  Accumulator columns per tile:
  // (verified for the 3-term bf16 stack, N = 96 / 192; the 2-term fp16 stack
  // at N = 64 / 256 lost the second term on B200 and stays one MMA per term)
  constexpr bool TSTACK = TERMS == 3 && BN <= 64;
  constexpr int ACC_N = TSTACK ? 3 * BN : BN;
  constexpr uint32_t TMEM_COLS = 2 * ACC_N <= 32 ? 32 : 2 * ACC_N <= 64 ? 64 : 2 * ACC_N <= 128 ? 128
                                 : 2 * ACC_N <= 256 ? 256 : 512;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *gbase = smem_raw + (base - raw);
  // ring addresses: A tile of k-block `it`, B tiles of stage s, bitmap ring
  constexpr uint32_t B_STRIDE = ABITS ? TERMS * B_BYTES : STAGE_BYTES;
  const uint32_t b_ring = base + (ABITS ? (uint32_t)kAStages * A_BYTES : A_BYTES);
  auto a_addr = [&](int it) -> uint32_t {
    return ABITS ? base + (uint32_t)(it % kAStages) * A_BYTES : base + (uint32_t)(it % stages) * STAGE_BYTES;
  };
  auto b_addr = [&](int s) -> uint32_t { return b_ring + (uint32_t)s * B_STRIDE; };
  const uint32_t bits_base = ABITS ? b_ring + (uint32_t)stages * B_STRIDE : 0u;
  const uint32_t bar0 = ABITS ? bits_base + (uint32_t)kBitsSlots * BITS_BYTES
                              : base + (uint32_t)stages * STAGE_BYTES;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (stages + s); };
  auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * stages + b); };
  auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * stages + 2 + b); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + (bar0 - base) + 8u * (2 * stages + 4));
  const uint32_t xbar0 = bar0 + 8u * (2 * stages + 4) + 16u;
  auto aready_bar = [&](int a) { return xbar0 + 8u * a; };  // leader: both CTAs' A tiles built
  auto aempty_bar = [&](int a) { return xbar0 + 8u * (kAStages + a); };  // multicast MMA commit
  auto bfull_bar = [&](int b) { return xbar0 + 8u * (2 * kAStages + b); };  // own CTA: bitmap landed
  auto bempty_bar = [&](int b) { return xbar0 + 8u * (2 * kAStages + kBitsSlots + b); };
  const uint32_t stage_c =
      (xbar0 + (ABITS ? 8u * (uint32_t)(2 * kAStages + 2 * kBitsSlots) : 0u) + 1023u) & ~1023u;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / 2, n_clusters = gridDim.x / 2;
  const int n_tiles_total = m_pairs * n_tiles;
  // this cluster's work items: the caller's LPT list, or round-robin tiles
  const bool sched = sarg.items != nullptr;
  const int t_begin = sched ? __ldg(sarg.cluster_start + cluster_id) : cluster_id;
  const int t_end = sched ? __ldg(sarg.cluster_start + cluster_id + 1) : n_tiles_total;
  const int t_step = sched ? 1 : n_clusters;
  auto item_at = [&](int i) {
    return sched ? __ldg(sarg.items + i) : make_int4(i, 0, -1, -1);
  };
  // every (step, k-block) this cluster reduces over, in the order all roles
  // walk them: fn(mp, st, kb), mp = the pair tile's first rank row
  auto walk = [&](auto &&fn) {
    for (int ti = t_begin; ti < t_end; ti += t_step) {
      const int4 item = item_at(ti);
      const int mp = (item.x / n_tiles) * (2 * BM);
      const int g_lo = item.y, g_hi = item.z < 0 ? INT32_MAX : item.z;
      int g = 0;
      for (int st = 0; st < sarg.n_steps && g < g_hi; ++st) {
        if (sarg.rows[st] <= mp) continue;
        for (int kb = 0; kb < sarg.nkb[st]; ++kb, ++g) {
          if (g < g_lo) continue;
          if (g >= g_hi) break;
          fn(mp, st, kb);
        }
      }
    }
  };

  if (warp == 1 && lane == 0) {
    for (int s = 0; s < sarg.n_steps; ++s)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a[s]))
                   : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int s = 0; s < stages; ++s) {
      // the leader's arrive.expect_tx calls (both CTAs' bytes; one per
      // producer warp) are the only arrivals: the peer's TMA bytes
      // complete_tx on the leader's barrier, and the peer cannot refill slot
      // s before the MMA that freed it has consumed this phase, so its bytes
      // never land in the wrong phase
      mbar_init(full_bar(s), ABITS ? 1 : 2);  // the leader's A and B producers
      mbar_init(empty_bar(s), 1);  // multicast MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    if constexpr (ABITS) {
      for (int a = 0; a < kAStages; ++a) {
        mbar_init(aready_bar(a), 8);  // 4 converter warps x 2 CTAs
        mbar_init(aempty_bar(a), 1);
      }
      for (int b = 0; b < kBitsSlots; ++b) {
        mbar_init(bfull_bar(b), 1);
        mbar_init(bempty_bar(b), 4);  // the consuming group's 4 warps
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // ---------------- TMA producers (both CTAs, whole warps) ----------------
  // A tiles (warp 0) and B tiles (warp 6; warp 0 when the converters build A)
  // stream from separate warps: a producer's per-k-block chain (empty wait,
  // expect_tx, tensor-map TMA issue) costs several hundred cycles of
  // mbarrier / TMA latency, and one producer for both operands was the
  // kernel's pace-setter (profiles/r01n_ncu_summary.md).  The leader's two
  // arrive.expect_tx are the full barrier's only arrivals (count 2).
  auto produce = [&](bool doA, bool doB) {
    const bool issuer = elect_one();
    int it = 0;
    for (int ti = t_begin; ti < t_end; ti += t_step) {
      const int4 item = item_at(ti);
      const int tile = item.x;
      const int mp = (tile / n_tiles) * (2 * BM);
      const int m0 = mp + (int)rank * BM;
      const int n0 = (tile % n_tiles) * BN + (int)rank * BH;
      const int g_lo = item.y, g_hi = item.z < 0 ? INT32_MAX : item.z;
      int g = 0;  // k-block index along the tile's step prefix
      for (int st = 0; st < sarg.n_steps && g < g_hi; ++st) {
        if (sarg.rows[st] <= mp) continue;  // pair-uniform: both CTAs load the same steps
        for (int kb = 0; kb < sarg.nkb[st]; ++kb, ++g) {
          if (g < g_lo) continue;
          if (g >= g_hi) break;
          const int s = it % stages;
          const int ph = ((it / stages) & 1) ^ 1;
          ++it;
          mbar_wait(empty_bar(s), ph);
          if (issuer) {
            const uint32_t lbar = mapa_shared(full_bar(s), 0);
            const bool la = !(sarg.dbg & 1) || kb == 0, lb = !(sarg.dbg & 2) || kb == 0;
            if (doA) {
              if (leader) mbar_expect_tx(full_bar(s), 2 * (la ? A_BYTES : 0));
              if (la) tma_load_2d_pair(a_addr(it - 1), &maps.a[st], lbar, kb * KB_EL, m0);  // rows >= rows[st]: zero fill
            }
            if (doB) {
              if (leader) mbar_expect_tx(full_bar(s), 2 * (lb ? TERMS * B_BYTES : 0));
              if (MNB) {  // one 3-D box: BH/64 feature blocks of 64 hub rows
                if (lb) tma_load_3d_pair(b_addr(s), &map_b, lbar, 0, sarg.c0[st] + kb * KB_EL, n0 / 64);
              } else {
#pragma unroll
                for (int q = 0; q < TERMS; ++q)
                  if (lb)
                    tma_load_2d_pair(b_addr(s) + q * B_BYTES, &map_b, lbar, sarg.c0[st] + kb * KB_EL,
                                     q * b_rows_per_term + n0);
              }
            }
          }
          __syncwarp();
        }
      }
    }
  };

  if (warp == 0) {
    produce(!ABITS, ABITS);
  } else if (!ABITS && warp == 6) {
    produce(false, true);
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, whole warp) ----------------
    // The loop runs warp-uniform so descriptors and TMEM addresses live in
    // uniform registers; one elected lane issues the MMAs and their commits
    // (a commit tracks the MMAs of the thread that issues it).  With a single
    // divergent lane every MMA cost a waterfall (ELECT / R2UR / BRA.U.ANY,
    // ~110 instructions per k-block) and the issue loop, not the tensor pipe,
    // set the pace (ncu: full barrier never waited on, tensor pipe 65 % busy).
    if (leader) {
      constexpr uint32_t idesc = FMT == 2 ? idesc_tf32_m256(ACC_N)
                                 : FMT == 4 ? idesc_f16_m256(ACC_N) | (1u << 16)  // B MN-major
                                 : FMT ? idesc_f16_m256(ACC_N) : idesc_bf16_m256(ACC_N);  // 1, 3: fp16
      const bool issuer = elect_one();
      int it = 0, lt = 0;
      for (int ti = t_begin; ti < t_end; ti += t_step, ++lt) {
        const int4 item = item_at(ti);
        const int tile = item.x;
        const int acc = lt & 1;
        mbar_wait(tempty_bar(acc), ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * ACC_N);
        const int kb_all = stair_kblocks(sarg, (tile / n_tiles) * (2 * BM));
        const int num_kb = (item.z < 0 ? kb_all : min(item.z, kb_all)) - item.y;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(full_bar(s), (it / stages) & 1);
          // converters of both CTAs wrote A with generic stores: cluster-scope acquire
          if constexpr (ABITS)
            if (!(sarg.dbg & 64)) mbar_wait_cluster(aready_bar(it % kAStages), (it / kAStages) & 1);
          tc_fence_after();
          // descriptor of k-step k = base + k * (32 B >> 4) in the start-address field
          const uint64_t ad0 = umma_desc_sw128(a_addr(it));
          // MN-major B: k-step k starts 16 rows (2 KB) further; K-major: 32 B further
          const uint64_t bd0 = MNB ? umma_desc_sw128_mn(b_addr(s), 8192) : umma_desc_sw128(b_addr(s));
          if (issuer && !(sarg.dbg & 4)) {
#pragma unroll
            for (int k = 0; k < KB_BYTES / MMA_K_BYTES; ++k) {
              const uint64_t ad = ad0 + (uint64_t)(k * (MMA_K_BYTES >> 4));
              if constexpr (TSTACK) {
                mma_bf16_pair(tmem_d, ad, bd0 + (uint64_t)(k * (MMA_K_BYTES >> 4)), idesc, (kb | k) != 0);
              } else {
#pragma unroll
                for (int q = 0; q < TERMS; ++q) {
                  const uint64_t bd = MNB ? bd0 + (uint64_t)((k * 16 * 128) >> 4)
                                          : bd0 + (uint64_t)((q * B_BYTES + k * MMA_K_BYTES) >> 4);
                  if constexpr (FMT == 2) mma_tf32_pair(tmem_d, ad, bd, idesc, (kb | k | q) != 0);
                  else mma_bf16_pair(tmem_d, ad, bd, idesc, (kb | k | q) != 0);
                }
              }
            }
          }
          if (issuer) {
            mma_commit_pair(empty_bar(s));  // frees slot s in both CTAs
            if constexpr (ABITS)
              if (!(sarg.dbg & 128)) mma_commit_pair(aempty_bar(it % kAStages));
          }
          __syncwarp();
        }
        if (issuer) mma_commit_pair(tfull_bar(acc));  // accumulators of both CTAs complete
        __syncwarp();
      }
    }
  } else if (ABITS && warp == 6) {  // ---------- bitmap producer (both CTAs) ----------
    if (lane == 0) {
      int it = 0;
      walk([&](int mp, int st, int kb) {
        const int b = it % kBitsSlots;
        mbar_wait(bempty_bar(b), ((it / kBitsSlots) & 1) ^ 1);
        ++it;
        // this CTA's 128 rows of the k-block's bitmap: 1 KB, contiguous
        const int rpad = (sarg.rows[st] + 255) & ~255;
        if (sarg.dbg & 32) {  // experiment: no bitmap traffic
          mbar_arrive(bfull_bar(b));
          return;
        }
        mbar_expect_tx(bfull_bar(b), BITS_BYTES);
        bulk_load_1d(bits_base + (uint32_t)b * BITS_BYTES,
                     sarg.bits[st] + (int64_t)kb * rpad + mp + (int)rank * BM, BITS_BYTES,
                     bfull_bar(b));
      });
    }
  } else if (ABITS && warp >= 7) {  // ---------- bitmap -> A tile converters (both CTAs) ----------
    // thread = tile row r: its 64-bit word becomes eight 16-byte chunks of
    // 16-bit ones/zeros, chunk c stored at (c ^ (r & 7)) — the SWIZZLE_128B
    // K-major layout TMA would have written
    const int r = ((warp - 7) & 3) * 32 + lane;
    const int grp = (warp - 7) >> 2;
    constexpr uint32_t ONE = FMT == 0 ? 0x3F80u : 0x3C00u;  // bf16 / fp16 1.0
    int it = 0;
    walk([&](int, int, int) {
      const int my = it++;
      if (my % kConvGroups != grp) return;
      const int b = my % kBitsSlots, a = my % kAStages;
      mbar_wait(bfull_bar(b), (my / kBitsSlots) & 1);
      if (!(sarg.dbg & 128)) mbar_wait(aempty_bar(a), ((my / kAStages) & 1) ^ 1);  // the MMA released A slot a
      const uint32_t sa = a_addr(my);
      uint64_t w;
      asm volatile("ld.shared.u64 %0, [%1];"
                   : "=l"(w)
                   : "r"(bits_base + (uint32_t)b * BITS_BYTES + (uint32_t)r * 8u)
                   : "memory");
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (sarg.dbg & 8) break;
        const uint32_t x = (uint32_t)(w >> (8 * c));
        uint32_t h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          h[j] = ((x >> (2 * j)) & 1u) * ONE | ((x >> (2 * j + 1)) & 1u) * (ONE << 16);
        const uint32_t dst = sa + (uint32_t)r * 128u + (uint32_t)((c ^ (r & 7)) * 16);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(h[0]), "r"(h[1]),
                     "r"(h[2]), "r"(h[3])
                     : "memory");
      }
      if (!(sarg.dbg & 16)) fence_proxy_async_smem();  // generic-proxy stores -> visible to the MMA
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bempty_bar(b));
        mbar_arrive_cluster(mapa_shared(aready_bar(a), 0));
      }
    });
  } else {  // ---------------- epilogue warps 2..5 (both CTAs) ----------------
    const int q = warp & 3;
    const bool relu = (ep.flags & GC_RELU) != 0;
    const bool accum = (ep.flags & GC_ACCUMULATE) != 0;
    const bool vec = ((ep.ldc & 3) == 0) && aligned16(ep.C);
    const uint32_t my_stage = stage_c + (uint32_t)(warp - 2) * 2u * 2048u;
    int lt = 0, sbuf = 0;
    for (int ti = t_begin; ti < t_end; ti += t_step, ++lt) {
      const int4 item = item_at(ti);
      const int tile = item.x;
      const int slot = item.w;
      const int acc = lt & 1;
      const int m0 = (tile / n_tiles) * (2 * BM) + (int)rank * BM;
      const int n0 = (tile % n_tiles) * BN;
      mbar_wait(tfull_bar(acc), (lt >> 1) & 1);
      tc_fence_after();
      const int rrow = m0 + q * 32 + lane;  // rank-ordered row
      const bool row_ok = rrow < ep.M;
      const int row = (row_ok && sarg.row_map) ? __ldg(sarg.row_map + rrow) : rrow;
      float rs = (row_ok && ep.row_scale) ? __ldg(ep.row_scale + row) : 1.0f;
      if (ep.scale) rs *= __ldg(ep.scale);
      float *crow = ep.C + (int64_t)row * ep.ldc;
      const uint32_t taddr = tmem_base + (uint32_t)(acc * ACC_N) + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        if (n0 + c >= ep.N) break;
        float v[16];
        if constexpr (TSTACK) {
          // feature chunk c lives in CTA half h at column j of each term group
          const int h = c / BH, jj = c % BH;
          float t1[16];
          tmem_ld16(taddr + (uint32_t)(h * TERMS * BH + jj), v);
#pragma unroll
          for (int q = 1; q < TERMS; ++q) {
            tmem_ld16(taddr + (uint32_t)(h * TERMS * BH + q * BH + jj), t1);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += t1[i];
          }
        } else {
          tmem_ld16(taddr + (uint32_t)c, v);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] *= rs;
          if (relu && !accum) v[i] = fmaxf(v[i], 0.0f);
        }
        if (sarg.dbg & 256) {  // experiment: no epilogue stores
          if (v[0] == 12345.678f) crow[0] = v[1];
          continue;
        }
        if (slot >= 0) {  // split-K partial: rank-row-major workspace tile, fixed up later
          if (row_ok) {
            float *w = sarg.ws + ((int64_t)slot * (2 * BM) + (int)rank * BM + q * 32 + lane) * BN + c;
#pragma unroll
            for (int i = 0; i < 16; i += 4) stg_f4(w + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
          }
          continue;
        }
        if (tma_store) {
          const uint32_t buf = my_stage + (uint32_t)sbuf * 2048u;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const uint32_t dst = buf + (uint32_t)lane * 64u + (uint32_t)((ch ^ ((lane >> 1) & 3)) * 16);
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "f"(v[4 * ch]),
                         "f"(v[4 * ch + 1]), "f"(v[4 * ch + 2]), "f"(v[4 * ch + 3])
                         : "memory");
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&map_c, buf, n0 + c, m0 + q * 32);
            bulk_commit();
          }
          sbuf ^= 1;
          continue;
        }
        if (!row_ok) continue;
        const int64_t col = n0 + c;
        if (accum) {
          if (vec && col + 16 <= ep.N) {  // 16-byte read-modify-write
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              float4 o = *reinterpret_cast<const float4 *>(crow + col + i);
              o.x += v[i], o.y += v[i + 1], o.z += v[i + 2], o.w += v[i + 3];
              if (relu) o.x = fmaxf(o.x, 0.f), o.y = fmaxf(o.y, 0.f), o.z = fmaxf(o.z, 0.f), o.w = fmaxf(o.w, 0.f);
              stg_f4(crow + col + i, o);
            }
            continue;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (col + i < ep.N) {
              float o = crow[col + i] + v[i];
              if (relu) o = fmaxf(o, 0.0f);
              crow[col + i] = o;
            }
          continue;
        }
        if (vec && col + 16 <= ep.N) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            stg_f4(crow + col + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (col + i < ep.N) crow[col + i] = v[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(tempty_bar(acc), 0));
    }
    if (tma_store && lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done (MMAs retired, epilogues drained)
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
}

template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tf32_tcgen05(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_c, const GemmEpi ep, int num_kb,
                      int stages, int m_tiles, int n_tiles, int tma_store) {
  gemm_tc_body<BN, 1, 0>(map_a, map_b, map_c, ep, num_kb, stages, m_tiles, n_tiles, tma_store, 0);
}

// 3xTF32 (fp32-class) dense update: B = [hi(W^T); lo(W^T)] (b_rows_per_term
// rows each), A split into hi / lo on chip (see gemm_tc_body SPLITA).
template <int BN>
__global__ void __launch_bounds__(kGemmThreads + kConvThreads, 1)
    gemm_tf32x3_tcgen05(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_c, const GemmEpi ep, int num_kb,
                        int stages, int m_tiles, int n_tiles, int tma_store, int b_rows_per_term) {
  gemm_tc_body<BN, 2, 0, true>(map_a, map_b, map_c, ep, num_kb, stages, m_tiles, n_tiles,
                               tma_store, b_rows_per_term);
}

// Dense hub block of the hybrid aggregation: C = D_row · A_hub · (B0 + B1 + B2)
// with A_hub the 0/1 adjacency restricted to the hub columns (exact in bf16)
// and B_q the three bf16 terms of D_col·X[hub rows] (together exact fp32).
template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_hub_bf16x3_tcgen05(const __grid_constant__ CUtensorMap map_a,
                            const __grid_constant__ CUtensorMap map_b,
                            const __grid_constant__ CUtensorMap map_c, const GemmEpi ep,
                            int num_kb, int stages, int m_tiles, int n_tiles, int tma_store,
                            int b_rows_per_term) {
  gemm_tc_body<BN, 3, 1>(map_a, map_b, map_c, ep, num_kb, stages, m_tiles, n_tiles, tma_store,
                         b_rows_per_term);
}

// One fp16 term of s·D·X (TF32-equivalent input rounding)
template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_hub_f16_tcgen05(const __grid_constant__ CUtensorMap map_a,
                         const __grid_constant__ CUtensorMap map_b,
                         const __grid_constant__ CUtensorMap map_c, const GemmEpi ep, int num_kb,
                         int stages, int m_tiles, int n_tiles, int tma_store, int b_rows_per_term) {
  gemm_tc_body<BN, 1, 2>(map_a, map_b, map_c, ep, num_kb, stages, m_tiles, n_tiles, tma_store,
                         b_rows_per_term);
}

// The same with the two-term FP16 split (hi/lo fp16 of s·D·X, s a power of two)
template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_hub_f16x2_tcgen05(const __grid_constant__ CUtensorMap map_a,
                           const __grid_constant__ CUtensorMap map_b,
                           const __grid_constant__ CUtensorMap map_c, const GemmEpi ep,
                           int num_kb, int stages, int m_tiles, int n_tiles, int tma_store,
                           int b_rows_per_term) {
  gemm_tc_body<BN, 2, 2>(map_a, map_b, map_c, ep, num_kb, stages, m_tiles, n_tiles, tma_store,
                         b_rows_per_term);
}

// W (K x N, ldw) -> Wt (N x K, ldt): the K-major B operand.  With Wt_lo
// (3xTF32): Wt = hi(W^T) (13 low mantissa bits cleared, exact in TF32) and
// Wt_lo = W^T - hi (exact in fp32).
__global__ void transpose_kernel(const float *__restrict__ W, int64_t ldw, int64_t K, int64_t N,
                                 float *__restrict__ Wt, int64_t ldt, float *__restrict__ Wt_lo) {
  __shared__ float tile[32][33];
  const int64_t k0 = (int64_t)blockIdx.y * 32, n0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t k = k0 + i, n = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && n < N) ? W[k * ldw + n] : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < ldt) {
      const float w = (k < K) ? tile[threadIdx.x][i] : 0.0f;
      if (Wt_lo) {
        const float hi = __uint_as_float(__float_as_uint(w) & 0xFFFFE000u);
        Wt[n * ldt + k] = hi;
        Wt_lo[n * ldt + k] = w - hi;
      } else {
        Wt[n * ldt + k] = w;
      }
    }
  }
}

// ============================================================================
// exact fp32 SIMT GEMM (64x64 tiles, 4x4 per thread, k ascending FMA)
// ============================================================================
constexpr int SB = 64, SK = 16;
__global__ void __launch_bounds__(256)
    gemm_fp32_simt(const float *__restrict__ A, int64_t lda, const float *__restrict__ W,
                   int64_t ldw, GemmEpi ep, int64_t K) {
  __shared__ float As[SK][SB + 4];
  __shared__ float Ws[SK][SB + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.x * SB, n0 = (int64_t)blockIdx.y * SB;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += SK) {
    for (int i = threadIdx.x; i < SB * SK; i += 256) {
      const int r = i / SK, kk = i % SK;  // A tile, read along k
      const int64_t gm = m0 + r, gk = k0 + kk;
      As[kk][r] = (gm < ep.M && gk < K) ? A[gm * lda + gk] : 0.0f;
      const int kr = i / SB, c = i % SB;  // W tile, read along n
      const int64_t wk = k0 + kr, wn = n0 + c;
      Ws[kr][c] = (wk < K && wn < ep.N) ? W[wk * ldw + wn] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + ty * 4 + i;
    if (r >= ep.M) continue;
    const float rs = ep.row_scale ? ep.row_scale[r] : 1.0f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = n0 + tx * 4 + j;
      if (c >= ep.N) continue;
      float v = acc[i][j] * rs;
      if (ep.flags & GC_RELU) v = fmaxf(v, 0.0f);
      ep.C[r * ep.ldc + c] = v;
    }
  }
}

__global__ void fill_rows_kernel(float *C, int64_t ldc, int64_t M, int64_t N, float v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M * N) C[(i / N) * ldc + i % N] = v;
}

// ============================================================================
// scale_rows / ReLU
// ============================================================================
__global__ void scale_rows_kernel(const float *__restrict__ d, const float *__restrict__ B,
                                  int64_t ldb, int64_t n_rows, int64_t K, float *__restrict__ C,
                                  int64_t ldc, uint32_t flags, bool vec) {
  const int64_t per_row = vec ? K / 4 : K;
  const int64_t total = n_rows * per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per_row, q = i % per_row;
    const float s = d ? __ldg(d + r) : 1.0f;
    if (vec) {
      float4 v = ldg_f4(B + r * ldb + 4 * q);
      v.x *= s, v.y *= s, v.z *= s, v.w *= s;
      if (flags & GC_RELU) {
        v.x = fmaxf(v.x, 0.f), v.y = fmaxf(v.y, 0.f), v.z = fmaxf(v.z, 0.f), v.w = fmaxf(v.w, 0.f);
      }
      stg_f4(C + r * ldc + 4 * q, v);
    } else {
      float v = B[r * ldb + q] * s;
      if (flags & GC_RELU) v = fmaxf(v, 0.f);
      C[r * ldc + q] = v;
    }
  }
}

// ============================================================================
// host side: tensor maps
// ============================================================================
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

// 2-D fp32 row-major matrix (rows x cols, ld elements) as a K-major TMA map
// with a (BK x box_rows) box and 128-byte swizzle; OOB elements read as 0.
int make_map(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
             int box_rows, int box_cols = BK,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, bool bf16 = false,
             bool f16 = false) {
  auto enc = get_encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return GC_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * (bf16 ? 2 : 4))};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                        : bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, const_cast<void *>(ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GC_ERR_CUDA;
  }
  return GC_OK;
}

// MN-major B for the one-term pair GEMM: fp16 Bm[T][kp] viewed as
// {64 features, T rows, kp/64 feature blocks} so ONE box {64, 64, nblk}
// lands nblk 8 KB SWIZZLE_128B blocks (the MN blocks of the descriptor, LBO
// 8 KB apart) per stage
int make_map_mn(CUtensorMap *map, const void *ptr, int64_t T, int64_t kp, int nblk) {
  auto enc = get_encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return GC_ERR_CUDA;
  }
  cuuint64_t dims[3] = {64, (cuuint64_t)T, (cuuint64_t)(kp / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)(kp * 2), 128};
  cuuint32_t box[3] = {64, 64, (cuuint32_t)nblk};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void *>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (MN-major B) failed (%d)", (int)r);
    return GC_ERR_CUDA;
  }
  return GC_OK;
}

// smem: the stage ring, its barriers and (when it fits) the 16 KB epilogue
// staging for TMA stores; returns the stage count (0: does not fit)
inline int ring_stages(size_t stage_bytes, bool staging, size_t *smem,
                       size_t max_ring = 227 * 1024, size_t fixed = 0, int max_st = 8) {
  const size_t cap = 227 * 1024;
  for (int st = max_st; st >= 2; --st) {
    if ((size_t)st * stage_bytes > max_ring && st > 2) continue;
    const size_t need =
        (((size_t)st * stage_bytes + fixed + 8 * (2 * st + 4) + 16 + 1023) & ~(size_t)1023) +
        (staging ? 4 * 2 * 2048 : 0) + 1024;
    if (need <= cap) {
      *smem = need;
      return st;
    }
  }
  return 0;
}

template <int BN>
int launch_tf32(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mc, int tma_store,
                const GemmEpi &ep, int64_t K, cudaStream_t st) {
  const int num_kb = (int)((K + BK - 1) / BK);
  constexpr int stage_bytes = BM * KB_BYTES + BN * KB_BYTES;
  size_t smem = 0;
  const int stages = ring_stages(stage_bytes, true, &smem, 190 * 1024);
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_tf32_tcgen05<BN>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (attr_err != cudaSuccess) {
    set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
    return GC_ERR_CUDA;
  }
  const int m_tiles = (int)((ep.M + BM - 1) / BM);
  const int n_tiles = (int)((ep.N + BN - 1) / BN);
  const int64_t tiles = (int64_t)m_tiles * n_tiles;
  const int grid = (int)(tiles < sm_count() ? tiles : sm_count());  // persistent: one CTA per SM
  gemm_tf32_tcgen05<BN><<<grid, kGemmThreads, smem, st>>>(ma, mb, mc, ep, num_kb, stages, m_tiles,
                                                          n_tiles, tma_store);
  return check_launch("gemm_tf32_tcgen05");
}

template <int BN>
int launch_tf32x3(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mc,
                  int tma_store, const GemmEpi &ep, int64_t K, int b_rows_per_term,
                  cudaStream_t st) {
  const int num_kb = (int)((K + BK - 1) / BK);
  constexpr int stage_bytes = 2 * BM * KB_BYTES + 2 * BN * KB_BYTES;
  size_t smem = 0;
  const int stages = ring_stages(stage_bytes, true, &smem, 196 * 1024, 8 * 8);
  if (stages < 2) {
    set_error("gc_gemm_f32: 3xTF32 ring does not fit shared memory");
    return GC_ERR_UNSUPPORTED;
  }
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_tf32x3_tcgen05<BN>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (attr_err != cudaSuccess) {
    set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
    return GC_ERR_CUDA;
  }
  const int m_tiles = (int)((ep.M + BM - 1) / BM);
  const int n_tiles = (int)((ep.N + BN - 1) / BN);
  const int64_t tiles = (int64_t)m_tiles * n_tiles;
  const int grid = (int)(tiles < sm_count() ? tiles : sm_count());
  gemm_tf32x3_tcgen05<BN><<<grid, kGemmThreads + kConvThreads, smem, st>>>(
      ma, mb, mc, ep, num_kb, stages, m_tiles, n_tiles, tma_store, b_rows_per_term);
  return check_launch("gemm_tf32x3_tcgen05");
}

template <int BN, int FMT>
int launch_hub(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mc, int tma_store,
               const GemmEpi &ep, int64_t T, int64_t kp, cudaStream_t st) {
  constexpr int TERMS = fmt_terms(FMT);
  const int num_kb = (int)((T + 63) / 64);
  constexpr int stage_bytes = BM * KB_BYTES + TERMS * BN * KB_BYTES;
  size_t smem = 0;
  int stages = tma_store ? ring_stages(stage_bytes, true, &smem) : 0;
  if (stages == 0) {  // no room for the staging buffers: direct stores
    tma_store = 0;
    stages = ring_stages(stage_bytes, false, &smem);
  }
  if (stages == 0) {
    set_error("gc_hub_gemm: tile does not fit shared memory");
    return GC_ERR_UNSUPPORTED;
  }
  auto kern = FMT == 3 ? gemm_hub_f16_tcgen05<BN>
              : FMT ? gemm_hub_f16x2_tcgen05<BN> : gemm_hub_bf16x3_tcgen05<BN>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (attr_err != cudaSuccess) {
    set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
    return GC_ERR_CUDA;
  }
  const int m_tiles = (int)((ep.M + BM - 1) / BM);
  const int n_tiles = (int)((ep.N + BN - 1) / BN);
  const int64_t tiles = (int64_t)m_tiles * n_tiles;
  const int grid = (int)(tiles < sm_count() ? tiles : sm_count());
  kern<<<grid, kGemmThreads, smem, st>>>(ma, mb, mc, ep, num_kb, stages, m_tiles, n_tiles,
                                         tma_store, (int)kp);
  return check_launch(FMT == 3 ? "gemm_hub_f16_tcgen05"
                      : FMT ? "gemm_hub_f16x2_tcgen05" : "gemm_hub_bf16x3_tcgen05");
}

// Split-K fixup: per split tile, sum its workspace partials in slot order and
// add them to C through the rank permutation (deterministic).
__global__ void hub_splitk_fixup_kernel(const float *__restrict__ ws, const int4 *__restrict__ fix,
                                        const int32_t *__restrict__ row_map, float *__restrict__ C,
                                        int64_t ldc, int64_t M, int64_t N, int n_tiles, int bn) {
  const int4 f = fix[blockIdx.x];
  const int64_t m0 = (int64_t)(f.x / n_tiles) * 256, n0 = (int64_t)(f.x % n_tiles) * bn;
  for (int idx = threadIdx.x; idx < 256 * bn; idx += blockDim.x) {
    const int r = idx / bn, c = idx % bn;
    const int64_t rrow = m0 + r, col = n0 + c;
    if (rrow >= M || col >= N) continue;
    float sum = 0.0f;
    for (int k = 0; k < f.z; ++k) sum += ws[((int64_t)(f.y + k) * 256 + r) * bn + c];
    const int64_t row = row_map ? row_map[rrow] : rrow;
    C[row * ldc + col] += sum;
  }
}

template <int BN, int FMT, bool ABITS = false>
int launch_hub_pair(const StairMaps &maps, const StairArgs &sarg, const CUtensorMap &mb,
                    const CUtensorMap &mc, int tma_store, const GemmEpi &ep, int64_t kp,
                    cudaStream_t st, int sched_clusters = 0) {
  // (bitmap variant: B-only stages + the A and bitmap rings and their barriers)
  constexpr int stage_bytes = (ABITS ? 0 : BM * KB_BYTES) + fmt_terms(FMT) * (BN / 2) * KB_BYTES;
  constexpr size_t fixed =
      ABITS ? (size_t)kAStages * (BM * KB_BYTES + 16) + (size_t)kBitsSlots * (BM * 8 + 16) : 0;
  size_t smem = 0;
  static const int stage_cap = [] {  // GNNC_HUB_STAGES caps the ring (experiments)
    const char *e = getenv("GNNC_HUB_STAGES");
    return e ? atoi(e) : 0;
  }();
  const int max_st = stage_cap >= 2 ? stage_cap : ABITS ? 12 : 8;
  int stages = tma_store ? ring_stages(stage_bytes, true, &smem, 227 * 1024, fixed, max_st) : 0;
  if (stages == 0) {
    tma_store = 0;
    stages = ring_stages(stage_bytes, false, &smem, 227 * 1024, fixed, max_st);
  }
  if (stages == 0) {
    set_error("gc_hub_gemm: pair tile does not fit shared memory");
    return GC_ERR_UNSUPPORTED;
  }
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_hub_pair_tcgen05<BN, FMT, ABITS>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (attr_err != cudaSuccess) {
    set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
    return GC_ERR_CUDA;
  }
  const int m_pairs = (int)((ep.M + 2 * BM - 1) / (2 * BM));
  const int n_tiles = (int)((ep.N + BN - 1) / BN);
  const int64_t tiles = (int64_t)m_pairs * n_tiles;
  // tiles are walked in rank order = descending reduction length, round-robin
  // over the clusters, unless the caller passed an LPT schedule
  const int clusters = sched_clusters > 0 ? sched_clusters
                                          : (int)(tiles < sm_count() / 2 ? tiles : sm_count() / 2);
  gemm_hub_pair_tcgen05<BN, FMT, ABITS><<<2 * clusters, ABITS ? kGemmThreads + kBitsThreads : kGemmThreads + 32,
                                         smem, st>>>(
      maps, mb, mc, ep, sarg, stages, m_pairs, n_tiles, tma_store, (int)kp);
  return check_launch("gemm_hub_pair_tcgen05");
}

inline int pair_bn(int64_t K) { return K <= 32 ? 32 : K <= 64 ? 64 : K <= 128 ? 128 : 256; }

template <int FMT, bool ABITS = false, typename... Args>
int launch_hub_pair_bn_f(int pbn, Args &&...args) {
  switch (pbn) {
    case 32: return launch_hub_pair<32, FMT, ABITS>(args...);
    case 64: return launch_hub_pair<64, FMT, ABITS>(args...);
    case 128: return launch_hub_pair<128, FMT, ABITS>(args...);
    default: return launch_hub_pair<256, FMT, ABITS>(args...);
  }
}
// the staircase with bit-packed A blocks (kind::f16 formats only)
template <typename... Args>
int launch_hub_pair_bits(int kfmt, int pbn, Args &&...args) {
  switch (kfmt) {
    case 3: return launch_hub_pair_bn_f<3, true>(pbn, args...);
    case 1: return launch_hub_pair_bn_f<1, true>(pbn, args...);
    default: return launch_hub_pair_bn_f<0, true>(pbn, args...);
  }
}
// kfmt: the kernel's FMT (0 bf16x3, 1 f16x2, 2 tf32, 3 f16) — see kernel_fmt()
template <typename... Args>
int launch_hub_pair_bn(int kfmt, int pbn, Args &&...args) {
  switch (kfmt) {
    case 2: return launch_hub_pair_bn_f<2>(pbn, args...);
    case 3: return launch_hub_pair_bn_f<3>(pbn, args...);
    case 4: return pbn >= 256 ? launch_hub_pair<256, 4>(args...) : launch_hub_pair<128, 4>(args...);
    case 1: return launch_hub_pair_bn_f<1>(pbn, args...);
    default: return launch_hub_pair_bn_f<0>(pbn, args...);
  }
}
template <int FMT, typename... Args>
int launch_hub_bn_f(int bn, Args &&...args) {
  switch (bn) {
    case 16: return launch_hub<16, FMT>(args...);
    case 32: return launch_hub<32, FMT>(args...);
    case 64: return launch_hub<64, FMT>(args...);
    case 128: return launch_hub<128, FMT>(args...);
    default: return launch_hub<256, FMT>(args...);
  }
}

// ABI term format (GC_HUB_*) -> kernel FMT, term count, 16-bit element kind
inline int kernel_fmt(int32_t fmt) {
  return fmt == GC_HUB_F16_MN ? 4 : fmt == GC_HUB_F16 ? 3 : fmt == GC_HUB_F16X2 ? 1 : 0;
}
inline int hub_terms(int32_t fmt) {
  return (fmt == GC_HUB_F16 || fmt == GC_HUB_F16_MN) ? 1 : fmt == GC_HUB_F16X2 ? 2 : 3;
}
inline bool hub_is_f16(int32_t fmt) { return fmt != GC_HUB_BF16X3; }
inline bool hub_fmt_ok(int32_t fmt) {
  return fmt == GC_HUB_BF16X3 || fmt == GC_HUB_F16X2 || fmt == GC_HUB_F16 || fmt == GC_HUB_F16_MN;
}

inline bool gemm_pair_enabled() {  // GNNC_GEMM_PAIR=0: TF32 GEMM on single CTAs
  static const bool on = [] {
    const char *e = getenv("GNNC_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

inline bool hub_pair_enabled() {
  static const bool on = [] {
    const char *e = getenv("GNNC_HUB_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// X[hub_cols[t], f] * d[hub_cols[t]] -> three bf16 terms, transposed to the
// K-major B operand Bt[q][f][t] (f < kp; rows f >= K are zero).  hi = bf16(x),
// mid = bf16(x - hi), lo = bf16(x - hi - mid): hi + mid + lo carries x's full
// 24-bit mantissa, so A_hub (0/1) · B is an fp32-exact product.
__device__ __forceinline__ void split3(float x, __nv_bfloat16 &hi, __nv_bfloat16 &mid,
                                       __nv_bfloat16 &lo) {
  hi = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r1);
  lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
}

// 64 hub rows x 32 features per block: coalesced 128-byte reads of the
// gathered rows, then each thread writes a bf16x2 pair of hub positions for
// each of the three terms (128-byte rows of the K-major operand per warp).
__global__ void __launch_bounds__(256)
    hub_pack_kernel(const float *__restrict__ X, int64_t ldx, int64_t K,
                    const int32_t *__restrict__ hub_cols, int64_t T,
                    const float *__restrict__ d, int64_t kp, __nv_bfloat16 *__restrict__ Bt) {
  __shared__ float tile[64][33];
  const int64_t t0 = (int64_t)blockIdx.x * 64, f0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 64; i += blockDim.y) {
    const int64_t t = t0 + i, f = f0 + threadIdx.x;
    float x = 0.0f;
    if (t < T && f < K) {
      const int64_t j = __ldg(hub_cols + t);
      x = __ldg(X + j * ldx + f);
      if (d) x *= __ldg(d + j);
    }
    tile[i][threadIdx.x] = x;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t f = f0 + i, t = t0 + 2 * threadIdx.x;
    if (f >= kp || t >= T) continue;
    __nv_bfloat16 h0, m0, l0, h1, m1, l1;
    split3(tile[2 * threadIdx.x][i], h0, m0, l0);
    split3(tile[2 * threadIdx.x + 1][i], h1, m1, l1);
    // T is a multiple of 64, so (t, t + 1) are both in range and 4-byte aligned
    *reinterpret_cast<__nv_bfloat162 *>(Bt + f * T + t) = __halves2bfloat162(h0, h1);
    *reinterpret_cast<__nv_bfloat162 *>(Bt + (kp + f) * T + t) = __halves2bfloat162(m0, m1);
    *reinterpret_cast<__nv_bfloat162 *>(Bt + (2 * kp + f) * T + t) = __halves2bfloat162(l0, l1);
  }
}

// scale chunk of feature f: 256-column chunks when sig_ld > 1, else the row's
__device__ __forceinline__ int64_t sig_chunk(int64_t f, int sig_ld) {
  return sig_ld > 1 ? (f >> 8) : 0;
}

// |(D X)[hub_cols]| maximum (as float bits; non-negative floats order like
// ints): a warp per gathered row, lanes across its K floats.
__global__ void __launch_bounds__(256)
    hub_absmax_kernel(const float *__restrict__ X, int64_t ldx, int64_t K,
                      const int32_t *__restrict__ hub_cols, int64_t T,
                      const float *__restrict__ d, unsigned *__restrict__ out,
                      const __half *__restrict__ Xh = nullptr,
                      const float *__restrict__ sigma = nullptr, int sig_ld = 1) {
  // Xh (fp16 rows, scales sigma) replaces X when given: x = sigma_j * Xh[j]
  // (sig_ld > 1: one scale per 256-column chunk, sigma[j * sig_ld + f / 256])
  const int lane = threadIdx.x % 32;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t n_warps = (int64_t)gridDim.x * blockDim.x / 32;
  float m = 0.0f;
  for (int64_t t = warp; t < T; t += n_warps) {
    const int64_t j = __ldg(hub_cols + t);
    float mr = 0.0f;
    if (Xh) {
      const __half *row = Xh + j * ldx;
      for (int64_t f = lane; f < K; f += 32)
        mr = fmaxf(mr, fabsf(__half2float(row[f]) * __ldg(sigma + j * sig_ld + sig_chunk(f, sig_ld))));
    } else {
      const float *row = X + j * ldx;
      for (int64_t f = lane; f < K; f += 32) mr = fmaxf(mr, fabsf(__ldg(row + f)));
    }
    m = fmaxf(m, d ? mr * fabsf(__ldg(d + j)) : mr);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomicMax(out, __float_as_uint(m));
}

// Two fp16 terms of s·x, s = 2^(13 - floor(log2 max|x|)) so max|s·x| < 2^14:
// hi = fp16(s x), lo = fp16(s x - hi) carry 22 significant bits of every
// element above 2^-10 max|x| (absolute error <= 2^-23 max|x| for all).
// TERMS == 1 writes hi only: 11 significant bits, TF32's input rounding.
// Block (0, 0) publishes 1/s in scale[1] for the GEMM epilogue.
template <int TERMS>
__global__ void __launch_bounds__(256)
    hub_pack_f16_kernel(const float *__restrict__ X, int64_t ldx, int64_t K,
                        const int32_t *__restrict__ hub_cols, int64_t T,
                        const float *__restrict__ d, int64_t kp, const unsigned *__restrict__ amax,
                        float *__restrict__ inv_scale, __half *__restrict__ Bt,
                        const __half *__restrict__ Xh = nullptr,
                        const float *__restrict__ sigma = nullptr, int sig_ld = 1) {
  __shared__ float tile[64][33];
  const float mx = __uint_as_float(*amax);
  const int e = mx > 0.0f ? ilogbf(mx) : 0;
  const float sc = ldexpf(1.0f, 13 - e);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    *inv_scale = ldexpf(1.0f, e - 13);
  const int64_t t0 = (int64_t)blockIdx.x * 64, f0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 64; i += blockDim.y) {
    const int64_t t = t0 + i, f = f0 + threadIdx.x;
    float x = 0.0f;
    if (t < T && f < K) {
      const int64_t j = __ldg(hub_cols + t);
      x = Xh ? __half2float(Xh[j * ldx + f]) * __ldg(sigma + j * sig_ld + sig_chunk(f, sig_ld))
             : __ldg(X + j * ldx + f);
      if (d) x *= __ldg(d + j);
    }
    tile[i][threadIdx.x] = x * sc;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t f = f0 + i, t = t0 + 2 * threadIdx.x;
    if (f >= kp || t >= T) continue;
    const float y0 = tile[2 * threadIdx.x][i], y1 = tile[2 * threadIdx.x + 1][i];
    const __half h0 = __float2half_rn(y0), h1 = __float2half_rn(y1);
    *reinterpret_cast<__half2 *>(Bt + f * T + t) = __halves2half2(h0, h1);
    if constexpr (TERMS == 2) {
      const __half l0 = __float2half_rn(y0 - __half2float(h0));
      const __half l1 = __float2half_rn(y1 - __half2float(h1));
      *reinterpret_cast<__half2 *>(Bt + (kp + f) * T + t) = __halves2half2(l0, l1);
    }
  }
}

// One fp16 term of s·x, rows as gathered ([T][kp], features contiguous: the
// MN-major B operand, no transpose).  Warp per hub row, 8 features per lane
// per pass (two float4 loads, one 16-byte store); features >= K are zero.
__global__ void __launch_bounds__(256)
    hub_pack_f16_mn_kernel(const float *__restrict__ X, int64_t ldx, int64_t K,
                           const int32_t *__restrict__ hub_cols, int64_t T,
                           const float *__restrict__ d, int64_t kp,
                           const unsigned *__restrict__ amax, float *__restrict__ inv_scale,
                           __half *__restrict__ Bm, int vec, const __half *__restrict__ Xh = nullptr,
                           const float *__restrict__ sigma = nullptr, int sig_ld = 1) {
  const float mx = __uint_as_float(*amax);
  const int e = mx > 0.0f ? ilogbf(mx) : 0;
  const float sc = ldexpf(1.0f, 13 - e);
  if (blockIdx.x == 0 && threadIdx.x == 0) *inv_scale = ldexpf(1.0f, e - 13);
  const int lane = threadIdx.x % 32;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; t < T; t += n_warps) {
    const int64_t j = __ldg(hub_cols + t);
    const float *row = X + j * ldx;
    const __half *hrow = Xh ? Xh + j * ldx : nullptr;
    const float s0 = d ? __ldg(d + j) * sc : sc;
    for (int64_t f = 8 * lane; f < kp; f += 256) {
      // (8 features never straddle a 256-column scale chunk)
      const float s = Xh ? s0 * __ldg(sigma + j * sig_ld + sig_chunk(f, sig_ld)) : s0;
      float v[8];
      if (Xh) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = f + i < K ? __half2float(hrow[f + i]) : 0.0f;
      } else if (vec && f + 8 <= K) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(row + f));
        const float4 b = __ldg(reinterpret_cast<const float4 *>(row + f + 4));
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = f + i < K ? __ldg(row + f + i) : 0.0f;
      }
      __half2 h[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(v[2 * i] * s, v[2 * i + 1] * s);
      *reinterpret_cast<uint4 *>(Bm + t * kp + f) = *reinterpret_cast<const uint4 *>(h);
    }
  }
}

inline int hub_bn(int64_t K) {
  static const int cap = [] {  // GNNC_HUB_BN caps the N tile (experiments)
    const char *e = getenv("GNNC_HUB_BN");
    const int v = e ? atoi(e) : 128;  // 128: 3-stage ring (measured faster than 256 x 2 stages)
    return (v == 16 || v == 32 || v == 64 || v == 128) ? v : 256;
  }();
  const int bn = K <= 16 ? 16 : K <= 32 ? 32 : K <= 64 ? 64 : K <= 128 ? 128 : 256;
  return bn < cap ? bn : cap;
}

}  // namespace
}  // namespace gnnc

using namespace gnnc;

extern "C" size_t gc_gemm_workspace_bytes(int64_t K, int64_t N) {
  if (K <= 0 || N <= 0) return 0;
  const int64_t ldt = (K + 3) / 4 * 4;
  return (size_t)(2 * N * ldt * 4);  // W^T, and its lo term for 3xTF32
}

extern "C" int gc_gemm_f32(const float *A, int64_t lda, const float *W, int64_t ldw, int64_t M,
                           int64_t K, int64_t N, float *C, int64_t ldc, const float *row_scale,
                           uint32_t flags, void *workspace, size_t ws_bytes, void *stream) {
  GC_REQUIRE(M >= 0 && K >= 0 && N >= 0, GC_ERR_SHAPE, "gc_gemm_f32: negative size");
  GC_REQUIRE(lda >= K && ldw >= N && ldc >= N, GC_ERR_SHAPE, "gc_gemm_f32: bad leading dim");
  const bool tf32 = (flags & GC_GEMM_TF32) != 0, fp32 = (flags & GC_GEMM_FP32) != 0;
  const bool x3 = (flags & GC_GEMM_TF32X3) != 0;
  GC_REQUIRE((int)tf32 + (int)fp32 + (int)x3 == 1, GC_ERR_VALUE,
             "gc_gemm_f32: exactly one of TF32 / TF32X3 / FP32 required");
  GC_REQUIRE((flags & ~(GC_RELU | GC_GEMM_TF32 | GC_GEMM_FP32 | GC_GEMM_TF32X3)) == 0,
             GC_ERR_VALUE, "gc_gemm_f32: unknown flags 0x%x", flags);
  if (M == 0 || N == 0) return GC_OK;
  GC_REQUIRE(C && (K == 0 || (A && W)), GC_ERR_VALUE, "gc_gemm_f32: null operand");
  cudaStream_t st = as_stream(stream);
  GemmEpi ep{C, ldc, row_scale, M, N, flags};
  if (K == 0) {  // empty inner dimension: relu(0 * s) = 0
    const int64_t total = M * N;
    fill_rows_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(C, ldc, M, N, 0.0f);
    return check_launch("fill_rows_kernel");
  }
  if (fp32) {
    GC_REQUIRE((M + SB - 1) / SB < INT32_MAX && (N + SB - 1) / SB < 65536, GC_ERR_SHAPE,
               "gc_gemm_f32: grid too large");
    dim3 grid((unsigned)((M + SB - 1) / SB), (unsigned)((N + SB - 1) / SB));
    gemm_fp32_simt<<<grid, 256, 0, st>>>(A, lda, W, ldw, ep, K);
    return check_launch("gemm_fp32_simt");
  }
  // TF32 / 3xTF32 tensor-core path
  GC_REQUIRE((lda % 4) == 0 && aligned16(A), GC_ERR_UNSUPPORTED,
             "gc_gemm_f32: TF32 path needs lda %% 4 == 0 and a 16-byte aligned A");
  GC_REQUIRE(M < (int64_t)INT32_MAX && K < (int64_t)INT32_MAX, GC_ERR_SHAPE,
             "gc_gemm_f32: dimension exceeds TMA range");
  const size_t need = gc_gemm_workspace_bytes(K, N);
  GC_REQUIRE(workspace && ws_bytes >= need && aligned16(workspace), GC_ERR_WORKSPACE,
             "gc_gemm_f32: TF32 path needs %zu workspace bytes (16-byte aligned)", need);
  const int64_t ldt = (K + 3) / 4 * 4;
  float *wt = static_cast<float *>(workspace);
  {
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)((ldt + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(W, ldw, K, N, wt, ldt,
                                                     x3 ? wt + N * ldt : nullptr);
    int rc = check_launch("transpose_kernel");
    if (rc) return rc;
  }
  int bn = 256;
  if (N <= 16) bn = 16;
  else if (N <= 32) bn = 32;
  else if (N <= 64) bn = 64;
  else if (N <= 128) bn = 128;
  CUtensorMap ma, mb, mc;
  int rc = make_map(&ma, A, M, K, lda, BM);
  if (rc) return rc;
  if (x3) {
    // 3xTF32: A split on chip, B = [hi; lo] stacked (N rows per term); N
    // tiles of at most 128 columns keep three 64 KB stages in shared memory
    bn = bn > 128 ? 128 : bn;
    rc = make_map(&mb, wt, 2 * N, K, ldt, bn);
    if (rc) return rc;
    int tma_store = ((ldc % 4) == 0 && aligned16(C)) ? 1 : 0;
    memset(&mc, 0, sizeof(mc));
    if (tma_store) {
      rc = make_map(&mc, C, M, N, ldc, 32, 16, CU_TENSOR_MAP_SWIZZLE_64B);
      if (rc) return rc;
    }
    switch (bn) {
      case 16: return launch_tf32x3<16>(ma, mb, mc, tma_store, ep, K, (int)N, st);
      case 32: return launch_tf32x3<32>(ma, mb, mc, tma_store, ep, K, (int)N, st);
      case 64: return launch_tf32x3<64>(ma, mb, mc, tma_store, ep, K, (int)N, st);
      default: return launch_tf32x3<128>(ma, mb, mc, tma_store, ep, K, (int)N, st);
    }
  }
  if (hub_pair_enabled() && gemm_pair_enabled() && N > 16 && M >= 2 * BM &&
      (K >= 512 || M >= (int64_t(1) << 20))) {
    // CTA pairs (M = 256 per MMA, each CTA stages half of the W tile): the
    // hub GEMM's pipeline with one TF32 operand pair (FMT 2).  Measured:
    // 169K x 1024 x 1024 0.79 -> 0.60 ms, 2.45M x 256 x 256 1.15 -> 0.93 ms;
    // the HBM-bound 233K x 256 x 256 stays on single CTAs (0.117 vs 0.131 ms)
    const int pbn = pair_bn(N);
    CUtensorMap mbp;
    rc = make_map(&mbp, wt, N, K, ldt, pbn / 2);
    if (rc) return rc;
    int tma_store = ((ldc % 4) == 0 && aligned16(C)) ? 1 : 0;
    memset(&mc, 0, sizeof(mc));
    if (tma_store) {
      rc = make_map(&mc, C, M, N, ldc, 32, 16, CU_TENSOR_MAP_SWIZZLE_64B);
      if (rc) return rc;
    }
    StairMaps maps;
    memset(&maps, 0, sizeof(maps));
    maps.a[0] = ma;
    StairArgs sarg{};
    sarg.n_steps = 1;
    sarg.rows[0] = (int)M;
    sarg.c0[0] = 0;
    sarg.nkb[0] = (int)((K + BK - 1) / BK);
    return launch_hub_pair_bn(2, pbn, maps, sarg, mbp, mc, tma_store, ep, (int64_t)0, st, 0);
  }
  rc = make_map(&mb, wt, N, K, ldt, bn);
  if (rc) return rc;
  // output through TMA stores when C's pitch allows it (16-B aligned rows)
  int tma_store = ((ldc % 4) == 0 && aligned16(C)) ? 1 : 0;
  memset(&mc, 0, sizeof(mc));
  if (tma_store) {
    rc = make_map(&mc, C, M, N, ldc, 32, 16, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  switch (bn) {
    case 16: return launch_tf32<16>(ma, mb, mc, tma_store, ep, K, st);
    case 32: return launch_tf32<32>(ma, mb, mc, tma_store, ep, K, st);
    case 64: return launch_tf32<64>(ma, mb, mc, tma_store, ep, K, st);
    case 128: return launch_tf32<128>(ma, mb, mc, tma_store, ep, K, st);
    default: return launch_tf32<256>(ma, mb, mc, tma_store, ep, K, st);
  }
}

namespace gnnc {
namespace {
__global__ void __launch_bounds__(256)
    zero_rows_kernel(float *__restrict__ C, int64_t ldc, const int32_t *__restrict__ rows,
                     int64_t n, int64_t K, bool vec) {
  const int lane = threadIdx.x % 32;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < n; i += n_warps) {
    float *c = C + (int64_t)__ldg(rows + i) * ldc;
    if (vec)
      for (int64_t f = 4 * lane; f < K; f += 128)
        *reinterpret_cast<float4 *>(c + f) = make_float4(0.f, 0.f, 0.f, 0.f);
    else
      for (int64_t f = lane; f < K; f += 32) c[f] = 0.f;
  }
}
}  // namespace
}  // namespace gnnc

extern "C" int gc_zero_rows(float *C, int64_t ldc, const int32_t *rows, int64_t n_rows, int64_t K,
                            void *stream) {
  GC_REQUIRE(n_rows >= 0 && K >= 0 && ldc >= K, GC_ERR_SHAPE, "gc_zero_rows: bad shape");
  if (n_rows == 0 || K == 0) return GC_OK;
  GC_REQUIRE(C && rows, GC_ERR_VALUE, "gc_zero_rows: null operand");
  const bool vec = (K % 4 == 0) && (ldc % 4 == 0) && aligned16(C);
  const int64_t blocks = std::min<int64_t>((n_rows + 7) / 8, (int64_t)sm_count() * 16);
  zero_rows_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(C, ldc, rows, n_rows, K, vec);
  return check_launch("zero_rows_kernel");
}

extern "C" int gc_scale_rows_f32(const float *d, const float *B, int64_t ldb, int64_t n_rows,
                                 int64_t K, float *C, int64_t ldc, uint32_t flags, void *stream) {
  GC_REQUIRE(n_rows >= 0 && K >= 0 && ldb >= K && ldc >= K, GC_ERR_SHAPE,
             "gc_scale_rows_f32: bad shape");
  GC_REQUIRE((flags & ~GC_RELU) == 0, GC_ERR_VALUE, "gc_scale_rows_f32: unknown flags");
  if (n_rows == 0 || K == 0) return GC_OK;
  GC_REQUIRE(B && C, GC_ERR_VALUE, "gc_scale_rows_f32: null operand");
  const bool vec = (K % 4 == 0) && (ldb % 4 == 0) && (ldc % 4 == 0) && aligned16(B) && aligned16(C);
  const int64_t work = n_rows * (vec ? K / 4 : K);
  const int64_t blocks = (work + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 16;
  scale_rows_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, as_stream(stream)>>>(
      d, B, ldb, n_rows, K, C, ldc, flags, vec);
  return check_launch("scale_rows_kernel");
}

extern "C" int64_t gc_hub_terms_rows(int64_t K) {
  if (K <= 0) return 0;
  const int bn = hub_bn(K);
  return (K + bn - 1) / bn * bn;
}

extern "C" int gc_hub_pack(const float *X, int64_t ldx, int64_t K, const int32_t *hub_cols,
                           int64_t T, const float *d_col, int32_t fmt, void *Bt, float *scale_ws,
                           void *stream) {
  GC_REQUIRE(K >= 1 && T >= 0 && ldx >= K, GC_ERR_SHAPE, "gc_hub_pack: bad shape");
  GC_REQUIRE(hub_fmt_ok(fmt), GC_ERR_VALUE, "gc_hub_pack: format %d", fmt);
  if (T == 0) return GC_OK;
  GC_REQUIRE(X && hub_cols && Bt && (fmt == GC_HUB_BF16X3 || scale_ws), GC_ERR_VALUE,
             "gc_hub_pack: null operand");
  const int64_t kp = gc_hub_terms_rows(K);
  GC_REQUIRE(T % 64 == 0, GC_ERR_SHAPE, "gc_hub_pack: T must be a multiple of 64");
  dim3 grid((unsigned)((T + 63) / 64), (unsigned)((kp + 31) / 32));
  GC_REQUIRE(grid.y < 65536, GC_ERR_SHAPE, "gc_hub_pack: K too large");
  cudaStream_t st = as_stream(stream);
  if (fmt == GC_HUB_BF16X3) {
    hub_pack_kernel<<<grid, dim3(32, 8), 0, st>>>(X, ldx, K, hub_cols, T, d_col, kp,
                                                  static_cast<__nv_bfloat16 *>(Bt));
    return check_launch("hub_pack_kernel");
  }
  unsigned *amax = reinterpret_cast<unsigned *>(scale_ws);
  if (cudaMemsetAsync(amax, 0, sizeof(unsigned), st) != cudaSuccess) {
    set_error("gc_hub_pack: %s", cudaGetErrorString(cudaGetLastError()));
    return GC_ERR_CUDA;
  }
  const int64_t blocks = std::min<int64_t>((T + 7) / 8, (int64_t)sm_count() * 8);
  hub_absmax_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, ldx, K, hub_cols, T, d_col, amax);
  int rc = check_launch("hub_absmax_kernel");
  if (rc) return rc;
  if (fmt == GC_HUB_F16_MN) {
    GC_REQUIRE(aligned16(Bt) && kp % 8 == 0, GC_ERR_UNSUPPORTED, "gc_hub_pack: Bt alignment");
    const int vec = (ldx % 4 == 0 && aligned16(X)) ? 1 : 0;
    const int64_t nb = std::min<int64_t>((T + 7) / 8, (int64_t)sm_count() * 16);
    hub_pack_f16_mn_kernel<<<(unsigned)nb, 256, 0, st>>>(X, ldx, K, hub_cols, T, d_col, kp, amax,
                                                         scale_ws + 1, static_cast<__half *>(Bt), vec);
    return check_launch("hub_pack_f16_mn_kernel");
  }
  if (fmt == GC_HUB_F16)
    hub_pack_f16_kernel<1><<<grid, dim3(32, 8), 0, st>>>(X, ldx, K, hub_cols, T, d_col, kp, amax,
                                                         scale_ws + 1, static_cast<__half *>(Bt));
  else
    hub_pack_f16_kernel<2><<<grid, dim3(32, 8), 0, st>>>(X, ldx, K, hub_cols, T, d_col, kp, amax,
                                                         scale_ws + 1, static_cast<__half *>(Bt));
  return check_launch("hub_pack_f16_kernel");
}

extern "C" int gc_gemm_f16rows_f32(const float *A, int64_t lda, const float *W, int64_t ldw,
                                   int64_t M, int64_t K, int64_t N, const float *row_scale,
                                   void *Xh, int64_t ldh, float *sigma, void *workspace,
                                   size_t ws_bytes, void *stream) {
  GC_REQUIRE(M >= 0 && K >= 1 && N >= 1 && lda >= K && ldw >= N, GC_ERR_SHAPE,
             "gc_gemm_f16rows_f32: bad shape");
  GC_REQUIRE((N <= 256 || N % 256 == 0) && ldh == (N + 7) / 8 * 8, GC_ERR_UNSUPPORTED,
             "gc_gemm_f16rows_f32: needs N <= 256 or a multiple of 256, and ldh = N rounded "
             "up to 8");
  if (M == 0) return GC_OK;
  GC_REQUIRE(A && W && Xh && sigma && aligned16(Xh), GC_ERR_VALUE,
             "gc_gemm_f16rows_f32: null or unaligned operand");
  GC_REQUIRE((lda % 4) == 0 && aligned16(A), GC_ERR_UNSUPPORTED,
             "gc_gemm_f16rows_f32: needs lda %% 4 == 0 and a 16-byte aligned A");
  GC_REQUIRE(M < (int64_t)INT32_MAX, GC_ERR_SHAPE, "gc_gemm_f16rows_f32: M exceeds TMA range");
  const size_t need = gc_gemm_workspace_bytes(K, N);
  GC_REQUIRE(workspace && ws_bytes >= need && aligned16(workspace), GC_ERR_WORKSPACE,
             "gc_gemm_f16rows_f32: needs %zu workspace bytes (16-byte aligned)", need);
  cudaStream_t st = as_stream(stream);
  const int64_t ldt = (K + 3) / 4 * 4;
  float *wt = static_cast<float *>(workspace);
  {
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)((ldt + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(W, ldw, K, N, wt, ldt, nullptr);
    int rc = check_launch("transpose_kernel");
    if (rc) return rc;
  }
  const int bn = N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  // one scale per row (N <= 256) or per 256-column chunk: sigma is M x sig_ld
  GemmEpi ep{nullptr, 0, row_scale, M, N, 0u, nullptr,
             static_cast<__half *>(Xh), ldh, sigma, N <= 256 ? 1 : (int)(N / 256)};
  CUtensorMap ma, mb, mc;
  int rc = make_map(&ma, A, M, K, lda, BM);
  if (rc) return rc;
  rc = make_map(&mb, wt, N, K, ldt, bn);
  if (rc) return rc;
  memset(&mc, 0, sizeof(mc));
  switch (bn) {
    case 16: return launch_tf32<16>(ma, mb, mc, 0, ep, K, st);
    case 32: return launch_tf32<32>(ma, mb, mc, 0, ep, K, st);
    case 64: return launch_tf32<64>(ma, mb, mc, 0, ep, K, st);
    case 128: return launch_tf32<128>(ma, mb, mc, 0, ep, K, st);
    default: return launch_tf32<256>(ma, mb, mc, 0, ep, K, st);
  }
}

extern "C" int gc_hub_pack_f16rows(const void *Xh, int64_t ldh, const float *sigma, int64_t K,
                                   const int32_t *hub_cols, int64_t T, const float *d_col,
                                   int32_t fmt, void *Bt, float *scale_ws, void *stream) {
  // GC_HUB_SIG_CHUNKS(c) in fmt: sigma holds c scales per row (256 columns each)
  const int sig_ld = (int)(((uint32_t)fmt >> 8) & 15u) + 1;
  fmt &= 0xff;
  GC_REQUIRE(K >= 1 && T >= 0 && ldh >= K, GC_ERR_SHAPE, "gc_hub_pack_f16rows: bad shape");
  GC_REQUIRE(sig_ld == 1 || (int64_t)sig_ld * 256 == K, GC_ERR_SHAPE,
             "gc_hub_pack_f16rows: %d scale chunks need K = %d", sig_ld, sig_ld * 256);
  GC_REQUIRE(fmt == GC_HUB_F16 || fmt == GC_HUB_F16_MN, GC_ERR_VALUE,
             "gc_hub_pack_f16rows: one-term fp16 formats only (format %d)", fmt);
  if (T == 0) return GC_OK;
  GC_REQUIRE(Xh && sigma && hub_cols && Bt && scale_ws, GC_ERR_VALUE,
             "gc_hub_pack_f16rows: null operand");
  GC_REQUIRE(T % 64 == 0, GC_ERR_SHAPE, "gc_hub_pack_f16rows: T must be a multiple of 64");
  const int64_t kp = gc_hub_terms_rows(K);
  cudaStream_t st = as_stream(stream);
  const __half *xh = static_cast<const __half *>(Xh);
  unsigned *amax = reinterpret_cast<unsigned *>(scale_ws);
  if (cudaMemsetAsync(amax, 0, sizeof(unsigned), st) != cudaSuccess) {
    set_error("gc_hub_pack_f16rows: %s", cudaGetErrorString(cudaGetLastError()));
    return GC_ERR_CUDA;
  }
  const int64_t blocks = std::min<int64_t>((T + 7) / 8, (int64_t)sm_count() * 8);
  hub_absmax_kernel<<<(unsigned)blocks, 256, 0, st>>>(nullptr, ldh, K, hub_cols, T, d_col, amax,
                                                      xh, sigma, sig_ld);
  int rc = check_launch("hub_absmax_kernel");
  if (rc) return rc;
  if (fmt == GC_HUB_F16_MN) {
    GC_REQUIRE(aligned16(Bt) && kp % 8 == 0, GC_ERR_UNSUPPORTED,
               "gc_hub_pack_f16rows: Bt alignment");
    const int64_t nb = std::min<int64_t>((T + 7) / 8, (int64_t)sm_count() * 16);
    hub_pack_f16_mn_kernel<<<(unsigned)nb, 256, 0, st>>>(nullptr, ldh, K, hub_cols, T, d_col, kp,
                                                         amax, scale_ws + 1,
                                                         static_cast<__half *>(Bt), 0, xh, sigma,
                                                         sig_ld);
    return check_launch("hub_pack_f16_mn_kernel");
  }
  dim3 grid((unsigned)((T + 63) / 64), (unsigned)((kp + 31) / 32));
  GC_REQUIRE(grid.y < 65536, GC_ERR_SHAPE, "gc_hub_pack_f16rows: K too large");
  hub_pack_f16_kernel<1><<<grid, dim3(32, 8), 0, st>>>(nullptr, ldh, K, hub_cols, T, d_col, kp,
                                                       amax, scale_ws + 1,
                                                       static_cast<__half *>(Bt), xh, sigma,
                                                       sig_ld);
  return check_launch("hub_pack_f16_kernel");
}

extern "C" int gc_hub_gemm(const void *A_hub, int64_t lda, int64_t n_rows, int64_t T,
                           const void *Bt, int64_t K, int32_t fmt, const float *scale_ws,
                           float *C, int64_t ldc, const float *d_row, uint32_t flags,
                           void *stream) {
  GC_REQUIRE(n_rows >= 0 && T >= 0 && K >= 1 && lda >= T && ldc >= K, GC_ERR_SHAPE,
             "gc_hub_gemm: bad shape");
  GC_REQUIRE(hub_fmt_ok(fmt), GC_ERR_VALUE, "gc_hub_gemm: format %d", fmt);
  GC_REQUIRE((flags & ~(GC_RELU | GC_ACCUMULATE)) == 0, GC_ERR_VALUE,
             "gc_hub_gemm: unknown flags 0x%x", flags);
  if (n_rows == 0) return GC_OK;
  GC_REQUIRE(A_hub && Bt && C && (fmt == GC_HUB_BF16X3 || scale_ws), GC_ERR_VALUE,
             "gc_hub_gemm: null operand");
  GC_REQUIRE(T % 64 == 0 && T > 0 && lda % 8 == 0 && aligned16(A_hub) && aligned16(Bt),
             GC_ERR_UNSUPPORTED,
             "gc_hub_gemm: needs T %% 64 == 0, lda %% 8 == 0, 16-byte aligned operands");
  GC_REQUIRE(n_rows < (int64_t)INT32_MAX && T < (int64_t)INT32_MAX, GC_ERR_SHAPE,
             "gc_hub_gemm: dimension exceeds TMA range");
  cudaStream_t st = as_stream(stream);
  const int terms = hub_terms(fmt);
  const int bn = hub_bn(K);
  const int64_t kp = gc_hub_terms_rows(K);
  CUtensorMap ma, mb, mc;
  int rc = make_map(&ma, A_hub, n_rows, T, lda, BM, 64, CU_TENSOR_MAP_SWIZZLE_128B, true,
                    hub_is_f16(fmt));
  if (rc) return rc;
  GemmEpi ep{C, ldc, d_row, n_rows, K, flags, hub_is_f16(fmt) ? scale_ws + 1 : nullptr};
  // accumulating epilogues read C back: direct stores
  int tma_store = ((ldc % 4) == 0 && aligned16(C) && !(flags & GC_ACCUMULATE)) ? 1 : 0;
  memset(&mc, 0, sizeof(mc));
  if (tma_store) {
    rc = make_map(&mc, C, n_rows, K, ldc, 32, 16, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  GC_REQUIRE(fmt != GC_HUB_F16_MN || gc_hub_f16_mn_supported(K), GC_ERR_UNSUPPORTED,
             "gc_hub_gemm: GC_HUB_F16_MN needs gc_hub_f16_mn_supported(K)");
  if (hub_pair_enabled() && K > 16 && kp % pair_bn(K) == 0) {
    // CTA pairs: N = pair_bn, each CTA stages pair_bn/2 rows of each B term;
    // the plain hub block is a one-step staircase
    const int pbn = pair_bn(K);
    CUtensorMap mbp;
    rc = fmt == GC_HUB_F16_MN
             ? make_map_mn(&mbp, Bt, T, kp, pbn / 128)
             : make_map(&mbp, Bt, terms * kp, T, T, pbn / 2, 64, CU_TENSOR_MAP_SWIZZLE_128B, true,
                        hub_is_f16(fmt));
    if (rc) return rc;
    StairMaps maps;
    memset(&maps, 0, sizeof(maps));
    maps.a[0] = ma;
    StairArgs sarg{};
    sarg.n_steps = 1;
    sarg.rows[0] = (int)n_rows;
    sarg.c0[0] = 0;
    sarg.nkb[0] = (int)(T / 64);
    sarg.row_map = nullptr;
    return launch_hub_pair_bn(kernel_fmt(fmt), pbn, maps, sarg, mbp, mc, tma_store, ep, kp, st, 0);
  }
  rc = make_map(&mb, Bt, terms * kp, T, T, bn, 64, CU_TENSOR_MAP_SWIZZLE_128B, true,
                hub_is_f16(fmt));
  if (rc) return rc;
  switch (kernel_fmt(fmt)) {
    case 3: return launch_hub_bn_f<3>(bn, ma, mb, mc, tma_store, ep, T, kp, st);
    case 1: return launch_hub_bn_f<1>(bn, ma, mb, mc, tma_store, ep, T, kp, st);
    default: return launch_hub_bn_f<0>(bn, ma, mb, mc, tma_store, ep, T, kp, st);
  }
}

extern "C" int gc_hub_stair_pair_bn(int64_t K) { return K > 0 ? pair_bn(K) : 0; }

extern "C" int gc_hub_f16_mn_supported(int64_t K) {
  return (hub_pair_enabled() && K > 64 && gc_hub_terms_rows(K) % pair_bn(K) == 0 &&
          gc_hub_terms_rows(K) % 8 == 0)
             ? 1 : 0;
}

extern "C" int gc_hub_stair_supported(int64_t K) {
  return (hub_pair_enabled() && K > 16 && gc_hub_terms_rows(K) % pair_bn(K) == 0) ? 1 : 0;
}

extern "C" int gc_hub_stair_gemm(const void *const *A_steps, const int64_t *step_rows,
                                 const int64_t *step_c0, const int64_t *step_width,
                                 int32_t n_steps, const int32_t *row_map, const int32_t *items,
                                 const int32_t *cluster_start, int32_t n_clusters,
                                 float *workspace, const int32_t *fixups, int32_t n_fixups,
                                 const void *Bt, int64_t T, int64_t K, int32_t fmt,
                                 const float *scale_ws, float *C, int64_t ldc, const float *d_row,
                                 uint32_t flags, void *stream) {
  GC_REQUIRE(hub_fmt_ok(fmt) && (fmt == GC_HUB_BF16X3 || scale_ws), GC_ERR_VALUE,
             "gc_hub_stair_gemm: format %d", fmt);
  GC_REQUIRE(n_steps >= 1 && n_steps <= kMaxSteps, GC_ERR_VALUE,
             "gc_hub_stair_gemm: 1..%d steps", kMaxSteps);
  GC_REQUIRE(K >= 1 && T > 0 && T % 64 == 0 && ldc >= K, GC_ERR_SHAPE,
             "gc_hub_stair_gemm: bad shape");
  GC_REQUIRE((flags & ~(GC_RELU | GC_ACCUMULATE | GC_HUB_A_BITS)) == 0, GC_ERR_VALUE,
             "gc_hub_stair_gemm: unknown flags 0x%x", flags);
  const bool abits = (flags & GC_HUB_A_BITS) != 0;
  flags &= ~GC_HUB_A_BITS;
  GC_REQUIRE(A_steps && step_rows && step_c0 && step_width && Bt && C, GC_ERR_VALUE,
             "gc_hub_stair_gemm: null operand");
  GC_REQUIRE(gc_hub_stair_supported(K), GC_ERR_UNSUPPORTED,
             "gc_hub_stair_gemm: K=%lld has no CTA-pair tile", (long long)K);
  GC_REQUIRE(aligned16(Bt), GC_ERR_UNSUPPORTED, "gc_hub_stair_gemm: Bt alignment");
  StairMaps maps;
  memset(&maps, 0, sizeof(maps));
  GC_REQUIRE((items == nullptr) == (cluster_start == nullptr), GC_ERR_VALUE,
             "gc_hub_stair_gemm: items and cluster_start go together");
  GC_REQUIRE(items == nullptr || (n_clusters >= 1 && n_clusters <= sm_count() / 2),
             GC_ERR_VALUE, "gc_hub_stair_gemm: 1..%d clusters", sm_count() / 2);
  GC_REQUIRE(n_fixups >= 0 && (n_fixups == 0 || (fixups && workspace && items)), GC_ERR_VALUE,
             "gc_hub_stair_gemm: split-K needs items, workspace and fixups");
  GC_REQUIRE(n_fixups == 0 || !(flags & GC_RELU), GC_ERR_VALUE,
             "gc_hub_stair_gemm: ReLU cannot follow split-K partials");
  GC_REQUIRE(workspace == nullptr || aligned16(workspace), GC_ERR_WORKSPACE,
             "gc_hub_stair_gemm: 16-byte aligned workspace required");
  StairArgs sarg{};
  sarg.n_steps = n_steps;
  sarg.row_map = row_map;
  sarg.items = reinterpret_cast<const int4 *>(items);
  sarg.cluster_start = cluster_start;
  sarg.ws = workspace;
  static const int dbg = [] {
    const char *e = getenv("GNNC_HUB_DBG");
    return e ? atoi(e) : 0;
  }();
  sarg.dbg = dbg;
  for (int s = 0; s < n_steps; ++s) {
    const int64_t r = step_rows[s], c0 = step_c0[s], w = step_width[s];
    GC_REQUIRE(r >= 1 && r < INT32_MAX && w > 0 && w % 64 == 0 && c0 % 64 == 0 && c0 + w <= T,
               GC_ERR_SHAPE, "gc_hub_stair_gemm: bad step %d", s);
    GC_REQUIRE(s == 0 || (r <= step_rows[s - 1] && c0 == step_c0[s - 1] + step_width[s - 1]),
               GC_ERR_SHAPE, "gc_hub_stair_gemm: steps must be a staircase");
    GC_REQUIRE(A_steps[s] && aligned16(A_steps[s]), GC_ERR_VALUE,
               "gc_hub_stair_gemm: step %d operand", s);
    if (abits) {
      sarg.bits[s] = static_cast<const uint64_t *>(A_steps[s]);
    } else {
      int rc = make_map(&maps.a[s], A_steps[s], r, w, w, BM, 64, CU_TENSOR_MAP_SWIZZLE_128B, true,
                        hub_is_f16(fmt));
      if (rc) return rc;
    }
    sarg.rows[s] = (int)r;
    sarg.c0[s] = (int)c0;
    sarg.nkb[s] = (int)(w / 64);
  }
  const int64_t kp = gc_hub_terms_rows(K);
  const int pbn = pair_bn(K);
  GC_REQUIRE(fmt != GC_HUB_F16_MN || (gc_hub_f16_mn_supported(K) && !abits), GC_ERR_UNSUPPORTED,
             "gc_hub_stair_gemm: GC_HUB_F16_MN needs gc_hub_f16_mn_supported(K) and 16-bit blocks");
  CUtensorMap mbp, mc;
  int rc = fmt == GC_HUB_F16_MN
               ? make_map_mn(&mbp, Bt, T, kp, pbn / 128)
               : make_map(&mbp, Bt, hub_terms(fmt) * kp, T, T, pbn / 2, 64,
                          CU_TENSOR_MAP_SWIZZLE_128B, true, hub_is_f16(fmt));
  if (rc) return rc;
  memset(&mc, 0, sizeof(mc));
  // rank-ordered rows scatter through row_map: direct stores
  const int tma_store = (row_map == nullptr && (ldc % 4) == 0 && aligned16(C) &&
                         !(flags & GC_ACCUMULATE)) ? 1 : 0;
  if (tma_store) {
    rc = make_map(&mc, C, step_rows[0], K, ldc, 32, 16, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  GemmEpi ep{C, ldc, d_row, step_rows[0], K, flags, hub_is_f16(fmt) ? scale_ws + 1 : nullptr};
  cudaStream_t st = as_stream(stream);
  rc = abits ? launch_hub_pair_bits(kernel_fmt(fmt), pbn, maps, sarg, mbp, mc, tma_store, ep, kp,
                                    st, items ? (int)n_clusters : 0)
              : launch_hub_pair_bn(kernel_fmt(fmt), pbn, maps, sarg, mbp, mc, tma_store, ep, kp, st,
                                   items ? (int)n_clusters : 0);
  if (rc || n_fixups == 0) return rc;
  const int n_tiles = (int)((K + pbn - 1) / pbn);
  hub_splitk_fixup_kernel<<<(unsigned)n_fixups, 256, 0, st>>>(
      workspace, reinterpret_cast<const int4 *>(fixups), row_map, C, ldc, step_rows[0], K,
      n_tiles, pbn);
  return check_launch("hub_splitk_fixup_kernel");
}
