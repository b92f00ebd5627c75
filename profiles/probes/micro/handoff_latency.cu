// Handoff latencies on B200 (sm_100a), one CTA pair:
//  (1) mbarrier ping-pong between two warps of one CTA (arrive -> try_wait)
//  (2) tcgen05.commit (no MMA in flight) -> mbarrier, waited by the issuing warp
//  (3) ping-pong across the cluster (remote arrive on the peer CTA's barrier)
// Each loop runs N round trips; prints cycles per round trip.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void arrive_cluster(uint32_t b) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint32_t rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__global__ void __cluster_dims__(2, 1, 1) k(int n, long long *out) {
  __shared__ __align__(8) uint64_t bars[4];
  __shared__ uint32_t tslot;
  const uint32_t b0 = smem_u32(&bars[0]), b1 = smem_u32(&bars[1]), b2 = smem_u32(&bars[2]);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(b0, 1); mbar_init(b1, 1); mbar_init(b2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const bool r0 = rank() == 0;
  // (1) intra-CTA ping-pong: warp 0 arrives b0, warp 1 waits b0 and arrives b1
  long long t0 = clock64();
  if (lane == 0 && warp < 2) {
    for (int i = 0; i < n; ++i) {
      if (warp == 0) { arrive(b0); wait(b1, i & 1); }
      else { wait(b0, i & 1); arrive(b1); }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  // (2) commit with nothing in flight, waited by the same thread
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b2) : "memory");
      wait(b2, i & 1);
    }
  }
  __syncthreads();
  long long t2 = clock64();
  // (3) cluster ping-pong: rank 0 arrives on rank 1's b0, rank 1 on rank 0's b1... use b0 (recv)
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t3 = clock64();
  // re-init b0/b1 phases: use fresh counters via separate parity (b0,b1 completed n phases each)
  if (threadIdx.x == 0) {
    const uint32_t peer_b0 = mapa(smem_u32(&bars[3]), r0 ? 1 : 0);
    const uint32_t my = smem_u32(&bars[3]);
    if (r0) {
      mbar_init(my, 1);
    } else {
      mbar_init(my, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  t3 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t my = smem_u32(&bars[3]);
    const uint32_t peer = mapa(my, r0 ? 1 : 0);
    for (int i = 0; i < n; ++i) {
      if (r0) { arrive_cluster(peer); wait_cluster(my, i & 1); }
      else { wait_cluster(my, i & 1); arrive_cluster(peer); }
    }
  }
  __syncthreads();
  long long t4 = clock64();
  if (threadIdx.x == 0 && r0 && blockIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t4 - t3;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot));
}

int main() {
  long long *d, h[3];
  cudaMalloc(&d, sizeof(h));
  const int n = 10000;
  for (int rep = 0; rep < 2; ++rep) {
    k<<<2, 64>>>(n, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"intra_cta_pingpong_cycles\": %.1f, \"commit_roundtrip_cycles\": %.1f, "
         "\"cluster_pingpong_cycles\": %.1f}\n", h[0] / (double)n, h[1] / (double)n, h[2] / (double)n);
  return 0;
}
