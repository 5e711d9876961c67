// Grid-wide synchronisation helpers of the persistent kernels (persistent.cu,
// draft_loop.cu): acquire / release flags and a watchdog spin.
#pragma once
#include <stdint.h>

namespace sb {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until *p >= target.  A watchdog turns a protocol bug into a trapped
// kernel (an error the host sees) instead of a hung GPU.
__device__ __noinline__ static void wait_geq(const unsigned* p, unsigned target) {
  if (ld_acquire_u32(p) >= target) return;
  const uint64_t t0 = globaltimer();
  while (ld_acquire_u32(p) < target) {
    __nanosleep(32);
    if (globaltimer() - t0 > 20000000000ull) __trap();  // 20 s
  }
}
}  // namespace sb
