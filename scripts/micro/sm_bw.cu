// Per-SM achievable HBM read bandwidth: G CTAs (one per SM) stream disjoint
// chunks with cp.async.bulk (TMA 1-D) into a smem ring, or with 16-byte LDGs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) ldg_kernel(const uint4* __restrict__ src, size_t per_cta, uint4* sink) {
  const uint4* p = src + blockIdx.x * per_cta;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = threadIdx.x; i < per_cta; i += 256 * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = i + u * 256 < per_cta ? __ldcs(p + i + u * 256) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc.x ^= v[u].x, acc.y ^= v[u].y, acc.z ^= v[u].z, acc.w ^= v[u].w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) bulk_kernel(const char* __restrict__ src, size_t per_cta, int chunk, int stages) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const char* p = src + blockIdx.x * per_cta;
  const int n = (int)(per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(s32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    uint32_t phase[16] = {0};
    auto issue = [&](int i) {
      const int s = i % stages;
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       s32(sm + (size_t)s * chunk)),
                   "l"(p + (size_t)i * chunk), "r"(chunk), "r"(s32(&bar[s]))
                   : "memory");
    };
    for (int i = 0; i < stages && i < n; ++i) issue(i);
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(done)
                     : "r"(s32(&bar[s])), "r"(phase[s]));
      phase[s] ^= 1;
      if (i + stages < n) issue(i + stages);
    }
  }
  __syncthreads();
}

int main() {
  const size_t total = (size_t)2 << 30;  // 2 GiB source
  char* src;
  uint4* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 64);
  cudaMemset(src, 1, total);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int Gs[] = {1, 4, 8, 16, 32, 74, 148};
  for (int G : Gs) {
    const size_t per = (size_t)8 << 20;  // 8 MiB per CTA
    float best_l = 1e9, best_b = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      ldg_kernel<<<G, 256>>>((const uint4*)src, per / 16, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best_l) best_l = ms;
      cudaEventRecord(e0);
      bulk_kernel<<<G, 128, smem>>>(src, per, 32768, 6);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best_b) best_b = ms;
    }
    printf("G=%3d  LDG %7.1f GB/s total (%6.1f per SM)   bulk-TMA %7.1f GB/s total (%6.1f per SM)\n", G,
           G * per / best_l / 1e6, per / best_l / 1e6, G * per / best_b / 1e6, per / best_b / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
