// Shared helpers for the gnnc sm_100a kernels: error state, launch
// accounting, vector loads and small warp utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "gnnc.h"

namespace gnnc {

// ---- error state (thread-local message, set by every failing entry point) --
void set_error(const char *fmt, ...);
void clear_error();
void count_launch(uint64_t n = 1);

#define GC_REQUIRE(cond, code, ...)  \
  do {                               \
    if (!(cond)) {                   \
      ::gnnc::set_error(__VA_ARGS__); \
      return (code);                 \
    }                                \
  } while (0)

// Check the launch that was just issued; counts it on success.
inline int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return GC_ERR_CUDA;
  }
  count_launch();
  return GC_OK;
}

__host__ __device__ inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ float4 ldg_f4(const float *p) {
  float4 r;
  asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// Gathers with explicit L1 policy: hub rows stay resident (evict_last), the
// long tail streams through without allocating (no_allocate).
__device__ __forceinline__ float4 ldg_f4_keep(const float *p) {
  float4 r;
  asm("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ldg_f4_stream(const float *p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p));
  return r;
}

// Streaming loads (cache-streaming policy: evict-first in L1 and L2) for
// data read exactly once per kernel (col_idx, values).
__device__ __forceinline__ int ldg_stream_i32(const int32_t *p) { return __ldcs(p); }
__device__ __forceinline__ float ldg_stream_f32(const float *p) { return __ldcs(p); }

__device__ __forceinline__ void stg_f4(float *p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

__device__ __forceinline__ float fma4_dot(float4 a, float4 b, float acc) {
  acc = fmaf(a.x, b.x, acc);
  acc = fmaf(a.y, b.y, acc);
  acc = fmaf(a.z, b.z, acc);
  acc = fmaf(a.w, b.w, acc);
  return acc;
}

template <int W>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, W);
  return v;
}

template <int W>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o, W));
  return v;
}

__device__ __forceinline__ float leaky(float e, float slope) { return e < 0.0f ? e * slope : e; }

}  // namespace gnnc
