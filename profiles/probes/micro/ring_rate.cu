// Producer/consumer mbarrier ring without data (B200): iterations per cycle
// for S stages, consumer releasing slots by (a) mbarrier.arrive or (b)
// tcgen05.commit (no MMA in flight).  Two lanes in two warps of one CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}

template <bool COMMIT>
__global__ void ring(int n, int S, long long *out) {
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {  // producer
    for (int i = 0; i < n; ++i) {
      const int s = i % S;
      wait(smem_u32(&empty[s]), ((i / S) & 1) ^ 1);
      arrive(smem_u32(&full[s]));
    }
  } else if (warp == 1 && lane == 0) {  // consumer
    for (int i = 0; i < n; ++i) {
      const int s = i % S;
      wait(smem_u32(&full[s]), (i / S) & 1);
      if (COMMIT)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&empty[s])) : "memory");
      else
        arrive(smem_u32(&empty[s]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot));
}

int main() {
  long long *d, h;
  cudaMalloc(&d, sizeof(h));
  const int n = 20000;
  printf("{");
  for (int commit = 0; commit < 2; ++commit)
    for (int S : {1, 2, 4, 6, 8}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (commit) ring<true><<<1, 64>>>(n, S, d); else ring<false><<<1, 64>>>(n, S, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      }
      cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("\"%s_S%d\": %.1f, ", commit ? "commit" : "arrive", S, h / (double)n);
    }
  printf("\"unit\": \"cycles per iteration\"}\n");
  return 0;
}
