// Cost of tcgen05.commit on B200: issue throughput of back-to-back commits
// (no MMA in flight) for cta_group::1 and cta_group::2 with a 0b11 multicast,
// and the time until the last commit's mbarrier arrival is visible.
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

__global__ void __cluster_dims__(2, 1, 1) k(int n, long long *out) {
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tslot;
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  const uint32_t b0 = smem_u32(&bars[0]), b1 = smem_u32(&bars[1]);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b0), "r"(n));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b1), "r"(n));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  if (threadIdx.x == 0 && r == 0) {
    t0 = clock64();
    for (int i = 0; i < n; ++i)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0) : "memory");
    t1 = clock64();
    wait(b0, 0);
    t2 = clock64();
    for (int i = 0; i < n; ++i)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(b1), "h"((uint16_t)0x3) : "memory");
    t3 = clock64();
    wait(b1, 0);
    t4 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3;
  }
  if (threadIdx.x == 0 && r == 1) wait(b1, 0);  // the peer's copy completes too
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" ::"r"(tslot));
}

int main() {
  long long *d, h[4];
  cudaMalloc(&d, sizeof(h));
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) {
    k<<<2, 64>>>(n, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"commit_g1_issue_cycles\": %.1f, \"commit_g1_drain_cycles\": %lld, "
         "\"commit_g2_mc_issue_cycles\": %.1f, \"commit_g2_mc_drain_cycles\": %lld}\n",
         h[0] / (double)n, h[1], h[2] / (double)n, h[3]);
  return 0;
}
