// tcgen05 / TMEM / TMA GEMM for the bf16 verify forward and draft step (K2).
//
//   Y[M, N] = X[M, K] . W[N, K]^T      (bf16 in, fp32 accumulate in TMEM)
//
// Decode-shaped problems have few tokens (M = b(k+1) = 2..72 at b <= 8) and
// wide weights, so the kernel is written swap-AB: the weight tile is the MMA
// A operand (128 weight rows = UMMA_M 128), the token tile is the B operand
// (UMMA_N = M rounded up to 16, <= 256), and the accumulator D[128 x TN] lives
// in TMEM (lane = weight row, column = token).  The weight stream is the
// roofline term, so the work is split *stream-K*: the (tile, 64-wide k-block)
// units are divided evenly over a persistent grid of 148 x {1,2} CTAs, which
// keeps every SM streaming regardless of how many 128-row tiles a matrix has.
// A tile split across CTAs is fixed up deterministically: every contributor
// writes its fp32 partial to its own slot and the last arriving CTA sums the
// slots in k order (bit-reproducible, independent of arrival order).
//
// Warp roles (192 threads): warp 0 = TMA producer (one elected lane),
// warp 1 = TMEM allocator + MMA issuer (one elected lane), warps 2..5 =
// epilogue (tcgen05.ld 32x32b: warp w owns TMEM lanes 32*(w%4)..+31).
// Operands are staged by TMA with 128B swizzle into a multi-stage mbarrier
// ring; tcgen05.commit releases a stage back to the producer.
#include <cuda.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace sb {

constexpr int TC_BM = 128;   // weight rows per tile (UMMA_M)
constexpr int TC_BK = 64;    // k per stage (one 128-byte swizzle row of bf16)
constexpr int TC_UK = 16;    // k per tcgen05.mma (kind::f16)
constexpr int TC_THREADS = 192;
constexpr int TC_MAX_TN = 256;
// Stream-K tile counters live at the head of the workspace in a FIXED-size
// region (every GEMM sharing the workspace must agree on where partials start,
// or one GEMM's partial slots would clobber another's self-resetting counters).
constexpr int TC_MAX_TILES = 16384;
constexpr size_t TC_CNT_BYTES = (size_t)TC_MAX_TILES * 4;

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// 16 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// K-major, 128B-swizzled smem matrix descriptor (8-row x 128B swizzle atoms,
// SBO = 1024 B between atoms, descriptor version 1 for sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=tn.
__host__ __device__ constexpr uint32_t make_idesc(int tn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(tn >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}

struct TcParams {
  int M, N, K;
  int tn;          // UMMA_N (tokens per tile)
  int n_tiles_n;   // ceil(N / 128)
  int n_tiles;     // n_tiles_n * m_tiles
  int kb;          // k-blocks per tile
  int grid;        // persistent CTAs
  int stages;
  int epi;
  void* y;
  float* part;     // [grid][2][tn][128] fp32 partial slots
  int* counters;   // [n_tiles]
};

// segment = maximal run of one tile's k-blocks inside a CTA's unit range
struct Seg {
  int tile, kb0, kb1;
};

__device__ __forceinline__ long long unit_begin(int c, const TcParams& p) {
  return (long long)c * ((long long)p.n_tiles * p.kb) / p.grid;
}
__device__ __forceinline__ int cta_of_unit(long long u, const TcParams& p) {
  // smallest c with unit_begin(c+1) > u
  long long U = (long long)p.n_tiles * p.kb;
  int c = (int)((u * p.grid) / U);
  while (c + 1 < p.grid && unit_begin(c + 1, p) <= u) ++c;
  while (c > 0 && unit_begin(c, p) > u) --c;
  return c;
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.f + __expf(-g)); }

// Epilogue of one accumulator column set held by thread `lane_row` (weight row
// n = n0 + lane_row) for tokens m0 + j.
__device__ __forceinline__ void epi_store(const TcParams& p, int n, int m, float v, int row_in_warp) {
  // NOTE: SILU handled by caller (needs a lane shuffle)
  if (p.epi == EPI_STORE)
    ((__nv_bfloat16*)p.y)[(size_t)m * p.N + n] = __float2bfloat16_rn(v);
  else if (p.epi == EPI_STORE_F32)
    ((float*)p.y)[(size_t)m * p.N + n] = v;
  else
    ((float*)p.y)[(size_t)m * p.N + n] += v;
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int tn = p.tn;
  const uint32_t a_bytes = TC_BM * TC_BK * 2;
  const uint32_t b_bytes = tn * TC_BK * 2;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  uint8_t* stage_base = smem;
  uint64_t* full = (uint64_t*)(smem + p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* tmem_full = empty + p.stages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 1);
  int* flag = (int*)(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < tn) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const long long u_begin = unit_begin(c, p), u_end = unit_begin(c + 1, p);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (long long u = u_begin; u < u_end;) {
        int tile = (int)(u / p.kb);
        int kb0 = (int)(u - (long long)tile * p.kb);
        int kb1 = (int)min((long long)p.kb, u_end - (long long)tile * p.kb);
        int n0 = (tile % p.n_tiles_n) * TC_BM;
        int m0 = (tile / p.n_tiles_n) * tn;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = stage_base + stage * stage_bytes;
          mbar_expect_tx(&full[stage], stage_bytes);
          tma_load_2d(sa, &map_w, &full[stage], kb * TC_BK, n0);
          tma_load_2d(sa + a_bytes, &map_x, &full[stage], kb * TC_BK, m0);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        u = (long long)tile * p.kb + kb1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      const uint32_t idesc = make_idesc(tn);
      int stage = 0;
      uint32_t phase = 0;
      int seg = 0;
      for (long long u = u_begin; u < u_end; ++seg) {
        int tile = (int)(u / p.kb);
        int kb0 = (int)(u - (long long)tile * p.kb);
        int kb1 = (int)min((long long)p.kb, u_end - (long long)tile * p.kb);
        mbar_wait(tmem_empty, (seg & 1) ^ 1);
        tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          uint32_t sa = smem_u32(stage_base + stage * stage_bytes);
          uint32_t sb = sa + a_bytes;
#pragma unroll
          for (int kk = 0; kk < TC_BK / TC_UK; ++kk) {
            uint64_t ad = sw128_desc(sa + kk * TC_UK * 2);
            uint64_t bd = sw128_desc(sb + kk * TC_UK * 2);
            tc_mma(tmem, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(tmem_full);
        u = (long long)tile * p.kb + kb1;
      }
    }
  } else {
    // ---------------- epilogue warps (128 threads)
    const int quad = warp & 3;            // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;     // weight row within the tile
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    const int first_tile = (int)(u_begin / p.kb);
    int seg = 0;
    for (long long u = u_begin; u < u_end; ++seg) {
      int tile = (int)(u / p.kb);
      int kb0 = (int)(u - (long long)tile * p.kb);
      int kb1 = (int)min((long long)p.kb, u_end - (long long)tile * p.kb);
      const bool whole = (kb0 == 0 && kb1 == p.kb);
      const int n0 = (tile % p.n_tiles_n) * TC_BM;
      const int m0 = (tile / p.n_tiles_n) * tn;
      const int n = n0 + row;
      mbar_wait(tmem_full, seg & 1);
      tc_fence_after();
      float* slot = nullptr;
      if (!whole) slot = p.part + ((size_t)c * 2 + (tile == first_tile ? 0 : 1)) * (size_t)tn * TC_BM;
      for (int j0 = 0; j0 < tn; j0 += 16) {
        float v[16];
        tmem_ld16(lane_addr + j0, v);
        if (!whole) {
#pragma unroll
          for (int j = 0; j < 16; ++j) slot[(size_t)(j0 + j) * TC_BM + row] = v[j];
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            int m = m0 + j0 + j;
            if (p.epi == EPI_SILU_MUL) {
              float other = __shfl_xor_sync(0xffffffffu, v[j], 1);
              if (!(lane & 1) && m < p.M && n + 1 < p.N)
                ((__nv_bfloat16*)p.y)[(size_t)m * (p.N / 2) + n / 2] = __float2bfloat16_rn(silu_f(v[j]) * other);
            } else if (m < p.M && n < p.N) {
              epi_store(p, n, m, v[j], lane);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tmem_empty);
      if (!whole) {
        // stream-K fixup: publish the partial, last contributor reduces in k order
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const long long tu0 = (long long)tile * p.kb, tu1 = tu0 + p.kb - 1;
        const int c_first = cta_of_unit(tu0, p), c_last = cta_of_unit(tu1, p);
        if (threadIdx.x == 64) {
          int old = atomicAdd(&p.counters[tile], 1);
          *flag = (old == c_last - c_first);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (*flag) {
          __threadfence();
          for (int j = 0; j < tn; ++j) {
            int m = m0 + j;
            float acc = 0.f;
            for (int cc = c_first; cc <= c_last; ++cc) {
              int first_of_cc = (int)(unit_begin(cc, p) / p.kb);
              const float* sl = p.part + ((size_t)cc * 2 + (tile == first_of_cc ? 0 : 1)) * (size_t)tn * TC_BM;
              acc += __ldcg(&sl[(size_t)j * TC_BM + row]);
            }
            if (p.epi == EPI_SILU_MUL) {
              float other = __shfl_xor_sync(0xffffffffu, acc, 1);
              if (!(lane & 1) && m < p.M && n + 1 < p.N)
                ((__nv_bfloat16*)p.y)[(size_t)m * (p.N / 2) + n / 2] = __float2bfloat16_rn(silu_f(acc) * other);
            } else if (m < p.M && n < p.N) {
              epi_store(p, n, m, acc, lane);
            }
          }
          if (threadIdx.x == 64) p.counters[tile] = 0;  // self-cleaning for the next launch / graph replay
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      u = (long long)tile * p.kb + kb1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

static int make_map(CUtensorMap* map, const void* base, int rows, int cols, int ld, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return SB_EUNSUPPORTED;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : SB_EINVAL;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int tn_for(int M) {
  int t = (M + 15) / 16 * 16;
  return t < 16 ? 16 : (t > TC_MAX_TN ? TC_MAX_TN : t);
}

struct TcPlan {
  int tn, n_tiles_n, m_tiles, n_tiles, kb, grid, stages, ctas_per_sm;
  size_t smem, part_bytes, cnt_bytes;
};

static TcPlan plan(int M, int N, int K) {
  TcPlan q;
  q.tn = tn_for(M);
  q.n_tiles_n = (N + TC_BM - 1) / TC_BM;
  q.m_tiles = (M + q.tn - 1) / q.tn;
  q.n_tiles = q.n_tiles_n * q.m_tiles;
  q.kb = (K + TC_BK - 1) / TC_BK;
  q.ctas_per_sm = q.tn >= 128 ? 1 : 2;
  size_t budget = q.ctas_per_sm == 2 ? 108 * 1024 : 200 * 1024;
  size_t stage = (size_t)(TC_BM + q.tn) * TC_BK * 2;
  q.stages = (int)((budget - 1024 - 256) / stage);
  if (q.stages > 8) q.stages = 8;
  if (q.stages < 2) q.stages = 2;
  q.smem = 1024 + (size_t)q.stages * stage + 256;
  long long units = (long long)q.n_tiles * q.kb;
  long long g = (long long)num_sms() * q.ctas_per_sm;
  q.grid = (int)(units < g ? units : g);
  q.part_bytes = (size_t)q.grid * 2 * q.tn * TC_BM * 4;
  q.cnt_bytes = TC_CNT_BYTES;
  return q;
}

int gemm_tc_init() {
  static int rc = -1;
  if (rc < 0) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    rc = (e == cudaSuccess) ? 0 : (int)e;
    num_sms();
    get_encode();
  }
  return rc;
}

bool gemm_tc_supported(const GemmArgs& a) {
  if (a.dtype != SB_BF16) return false;
  if (a.K % 8 || a.ldx % 8) return false;  // 16-byte TMA strides
  if (((uintptr_t)a.x & 15) || ((uintptr_t)a.w & 15)) return false;
  if (a.epi == EPI_SILU_MUL && (a.N & 1)) return false;
  return get_encode() != nullptr;
}

size_t gemm_workspace_bytes(int M, int N, int K) {
  // sized for the simt fallback (none) and the tcgen05 stream-K partials
  const int tn = tn_for(M);
  size_t grid = (size_t)num_sms() * 2;
  return grid * 2 * tn * TC_BM * 4 + TC_CNT_BYTES + 4096;
}

int gemm_tc(const GemmArgs& a, cudaStream_t st) {
  if (!gemm_tc_supported(a)) return SB_EUNSUPPORTED;
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return SB_EINVAL;
  TcPlan q = plan(a.M, a.N, a.K);
  if (q.n_tiles > TC_MAX_TILES) return SB_EUNSUPPORTED;
  if (q.part_bytes + q.cnt_bytes > a.ws_bytes || !a.workspace) return SB_EWORKSPACE;
  CUtensorMap mw, mx;
  SB_TRY(make_map(&mw, a.w, a.N, a.K, a.K, TC_BM));
  SB_TRY(make_map(&mx, a.x, a.M, a.K, a.ldx, q.tn));
  TcParams p;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.tn = q.tn;
  p.n_tiles_n = q.n_tiles_n;
  p.n_tiles = q.n_tiles;
  p.kb = q.kb;
  p.grid = q.grid;
  p.stages = q.stages;
  p.epi = a.epi;
  p.y = a.y;
  p.counters = (int*)a.workspace;
  p.part = (float*)((char*)a.workspace + q.cnt_bytes);
  SB_TRY(gemm_tc_init());
  gemm_tc_kernel<<<q.grid, TC_THREADS, q.smem, st>>>(mw, mx, p);
  g_kernel_count++;
  SB_CHECK_LAUNCH();
  return 0;
}

}  // namespace sb
