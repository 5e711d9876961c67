// Shared device helpers for the specbatch_b200 kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "specbatch_b200.h"

#define SB_CHECK_LAUNCH()                              \
  do {                                                 \
    cudaError_t e_ = cudaGetLastError();               \
    if (e_ != cudaSuccess) return (int)e_;             \
  } while (0)

#define SB_TRY(expr)                \
  do {                              \
    int rc_ = (expr);               \
    if (rc_ != 0) return rc_;       \
  } while (0)

namespace sb {

extern thread_local int g_kernel_count;  // launches issued by the current forward
extern int g_pdl;                        // launch with programmatic stream serialization (PDL)

// Programmatic dependent launch: every kernel of the engine waits for its
// predecessor's memory before touching activations, and immediately lets its
// successor launch (the successor's prologue / weight prefetch overlaps).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Diagnostics (sb_debug_cta_trace): per-CTA timeline records of the traced kernels.
// buf[0] = record count (atomic); record r at buf + 8 + 8 r:
//   {launch id | kind << 32 | smid << 40, linear block id, t_entry, t_dependency_resolved,
//    t_first_stage (first operands on chip), t_mainloop_done, t_exit, 0}   (globaltimer ns)
extern unsigned long long* g_cta_trace;  // NULL = off
extern int g_cta_trace_seq;
extern int g_gemm_pre_max, g_gemm_launch_late, g_gemm_dbg;              // launch ids since the last sb_debug_cta_trace call
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cta_trace_write(unsigned long long* buf, int id, int kind, const unsigned long long* t) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const unsigned long long now = gtime();
  const unsigned long long r = atomicAdd(buf, 1ull);
  unsigned long long* o = buf + 8 + 8 * r;
  o[0] = (unsigned long long)(unsigned)id | ((unsigned long long)kind << 32) | ((unsigned long long)smid << 40);
  o[1] = blockIdx.x + (unsigned long long)gridDim.x * (blockIdx.y + (unsigned long long)gridDim.y * blockIdx.z);
  o[2] = t[0];
  o[3] = t[1];
  o[4] = t[2];
  o[5] = t[3];
  o[6] = now;
  o[7] = kind == 1 ? t[4] : 0;
}

// Launch helper: cudaLaunchKernelEx with the PDL attribute (and optional cluster).
template <typename... KArgs, typename... Args>
inline int launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
  if (e != cudaSuccess) return (int)e;
  ++g_kernel_count;
  return 0;
}

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (value, index) argmax with ties -> lowest index; NaN never wins.
struct ArgMax {
  float v;
  int i;
};
__device__ __forceinline__ ArgMax argmax_merge(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b{__shfl_xor_sync(0xffffffffu, a.v, o), __shfl_xor_sync(0xffffffffu, a.i, o)};
    a = argmax_merge(a, b);
  }
  return a;
}

// splitmix-style mix shared with the reference's `_mix` (engine.py:89-97) and
// with oracle/spec_ref.py: the counter RNG of the engine.
__host__ __device__ __forceinline__ uint64_t mix3(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t x = a * 0x9E3779B97F4A7C15ull + b * 0xBF58476D1CE4E5B9ull + c * 0x94D049BB133111EBull;
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
__host__ __device__ __forceinline__ float u01(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return (float)(mix3(seed, stream, ctr) >> 40) * (1.0f / 16777216.0f);
}


inline int grid_for(long n, int per_block, int cap = 148 * 16) {
  long g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace sb
