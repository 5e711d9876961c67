// Small-token GEMM (the draft model's decode step: T <= 16 tokens, K <= 3072): Y = X W^T with the
// fused-RMSNorm consumer / producer epilogues of the tcgen05 GEMM (gemm_tc.cu), for shapes where that
// kernel's fixed costs (TMEM allocation, barrier setup, cluster split-K reduction through DSMEM)
// dominate: a 68M draft step is ~10 such GEMMs of 1-5 MB of weights each.
//
// One CTA owns 16 (or 32) weight rows (m16n8k16 A tiles) and every token (B = X^T, n-tiles of 8 tokens);
// its 8 warps split K (32*C columns each), and the 8 partial tiles are summed through shared memory in
// warp order (deterministic).  Each lane loads 16 contiguous bytes of a weight row per 32-column chunk;
// the k order inside a chunk is permuted identically for A and B (dot products do not depend on it):
// physical columns 8t + 4s + {0,1 | 2,3} of chunk step s are the fragment's logical {2t,2t+1 | 2t+8,2t+9}.
// The warp's whole weight slice is loaded into registers BEFORE griddepcontrol.wait -- weights do not
// depend on the previous kernel -- so under PDL it streams while the producer of X still runs.
//
// Reference: the draft step is the reference's `ssm.step` (engine.py:138-145), charged as
// s * ssm_step_time (engine.py:196-198); this is the bf16 GEMM inside it.
#include "common.cuh"
#include "kernels.cuh"
#include "mma_ptx.cuh"

namespace sb {

constexpr int SG_W = 8;        // warps per CTA (K split)
constexpr int SG_TS = 20;      // shared row stride (floats) of a token's 16 partial rows: conflict-free
int g_small_gemm = 1;          // sb_set_small_gemm

struct SmallParams {
  const __nv_bfloat16* x;
  const __nv_bfloat16* w;
  void* y;
  int M, N, K, ldx;
  const float* ns_part;
  int ns_P, ns_stride;
  float ns_eps, ns_inv_h;
  float* out_part;
  __nv_bfloat16* out_xb;
  const __nv_bfloat16* out_gain;
  unsigned long long* trace;
  int trace_id;
};

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t u4_at(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ float silu_small(float g) { return __fdividef(g, 1.f + __expf(-g)); }

template <int E_, int C, int NT, int MT>
__global__ void __launch_bounds__(SG_W * 32, 1) gemm_small_kernel(SmallParams p) {
  __shared__ __align__(16) float red[SG_W][MT][16 * SG_TS];
  __shared__ float rs[16];
  __shared__ unsigned long long tr_t[5];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n0 = blockIdx.x * 16 * MT;
  const int kw0 = warp * 32 * C;
  if (p.trace && threadIdx.x == 0) {
    tr_t[0] = gtime();
    tr_t[4] = 0;
  }
  // the warp's weight slice: rows n0+16mt+g and +8, 16 bytes per chunk each
  uint4 a[MT][C][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        a[mt][c][h] = ldg_nc_v4(p.w + (size_t)(n0 + 16 * mt + g + 8 * h) * p.K + kw0 + 32 * c + 8 * t);
  // epilogue ownership: thread e -> token e/8, rows 2*(e%8), +1 of every m-tile (8 consecutive lanes)
  const int m = threadIdx.x >> 3, rp = threadIdx.x & 7;
  const bool mv = m < p.M && m < 8 * NT;
  float2 gain[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    gain[mt] = make_float2(1.f, 1.f);
    if (E_ == EPI_RESID_ADD && p.out_gain) {
      const int n = n0 + 16 * mt + 2 * rp;
      gain[mt] = make_float2(__bfloat162float(p.out_gain[n]), __bfloat162float(p.out_gain[n + 1]));
    }
  }
  griddep_wait();
  griddep_launch();
  if (p.trace && threadIdx.x == 0) tr_t[1] = gtime();
  // the residual rows this thread updates (final once the previous kernel completed): loaded now, used last
  float2 old[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
    old[mt] = (E_ == EPI_RESID_ADD && mv) ? __ldcg(reinterpret_cast<const float2*>((const float*)p.y + (size_t)m * p.N + n0 + 16 * mt + 2 * rp))
                                          : make_float2(0.f, 0.f);
  // consumer RMSNorm: 1/rms per token from the producer's partial sums (warp w: tokens w, w+8)
  if (p.ns_part) {
    for (int mm = warp; mm < p.M; mm += SG_W) {
      float s = 0.f;
      for (int q = lane; q < p.ns_P; q += 32) s += __ldcg(p.ns_part + (size_t)q * p.ns_stride + mm);
      s = warp_sum(s);
      if (lane == 0) rs[mm] = rsqrtf(s * p.ns_inv_h + p.ns_eps);
    }
  }
  if (p.trace && threadIdx.x == 0) tr_t[2] = gtime();
  float acc[MT][NT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[mt][nt][i] = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    uint4 b[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int mm = 8 * nt + g;
      b[nt] = mm < p.M ? ldg_nc_v4(p.x + (size_t)mm * p.ldx + kw0 + 32 * c + 8 * t) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          mma_bf16(acc[mt][nt], u4_at(a[mt][c][0], 2 * s), u4_at(a[mt][c][1], 2 * s), u4_at(a[mt][c][0], 2 * s + 1),
                   u4_at(a[mt][c][1], 2 * s + 1), u4_at(b[nt], 2 * s), u4_at(b[nt], 2 * s + 1));
  }
  // partial tiles -> shared: [warp][m-tile][token][row]
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    float* rw = red[warp][mt];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int tok = 8 * nt + 2 * t;
      rw[tok * SG_TS + g] = acc[mt][nt][0];
      rw[(tok + 1) * SG_TS + g] = acc[mt][nt][1];
      rw[tok * SG_TS + g + 8] = acc[mt][nt][2];
      rw[(tok + 1) * SG_TS + g + 8] = acc[mt][nt][3];
    }
  }
  __syncthreads();
  if (p.trace && threadIdx.x == 0) tr_t[3] = gtime();
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int n = n0 + 16 * mt + 2 * rp;
    float v0 = 0.f, v1 = 0.f;
    if (mv) {
#pragma unroll
      for (int w = 0; w < SG_W; ++w) {
        const float2 pr = *reinterpret_cast<const float2*>(&red[w][mt][m * SG_TS + 2 * rp]);
        v0 += pr.x;
        v1 += pr.y;
      }
      if (p.ns_part) {
        v0 *= rs[m];
        v1 *= rs[m];
      }
    }
    if (E_ == EPI_STORE) {
      if (mv) __stcs(reinterpret_cast<uint32_t*>((__nv_bfloat16*)p.y + (size_t)m * p.N + n), pack_bf16(v0, v1));
    } else if (E_ == EPI_SILU_MUL) {  // rows (n, n+1) = (gate, up)
      if (mv) __stcs((unsigned short*)p.y + (size_t)m * (p.N / 2) + n / 2,
                     __bfloat16_as_ushort(__float2bfloat16_rn(silu_small(v0) * v1)));
    } else {  // EPI_RESID_ADD: new residual, its bf16 copy scaled by the consumer's gain, norm partial
      const float a0 = old[mt].x + v0, a1 = old[mt].y + v1;
      if (mv) {
        __stcs(reinterpret_cast<float2*>((float*)p.y + (size_t)m * p.N + n), make_float2(a0, a1));
        if (p.out_xb)
          __stcs(reinterpret_cast<uint32_t*>(p.out_xb + (size_t)m * p.N + n), pack_bf16(a0 * gain[mt].x, a1 * gain[mt].y));
      }
      if (p.out_part) {
        float sq = mv ? a0 * a0 + a1 * a1 : 0.f;
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        sq += __shfl_xor_sync(0xffffffffu, sq, 4);
        if (mv && rp == 0) __stcs(p.out_part + (size_t)(blockIdx.x * MT + mt) * p.M + m, sq);
      }
    }
  }
  if (p.trace) {
    __syncthreads();
    if (threadIdx.x == 0) cta_trace_write(p.trace, p.trace_id, 1, tr_t);
  }
}

bool gemm_small_ok(const GemmArgs& a) {
  if (!g_small_gemm || a.dtype != SB_BF16) return false;
  if (a.M < 1 || a.M > 16 || a.N % 16 || a.K % 256 || a.K > 3072 || a.ldx % 8) return false;
  const int c = a.K / 256;
  if (!(c == 1 || c == 2 || c == 3 || c == 4 || c == 6 || c == 8 || c == 12)) return false;
  if (a.epi != EPI_STORE && a.epi != EPI_SILU_MUL && a.epi != EPI_RESID_ADD) return false;
  if (a.bias || a.relu || a.ln_s1 || a.ln_c1 || a.out_part1 || a.aux_val) return false;
  if (a.ns_part && (a.ns_row_step != 1 || a.ns_row_off != 0)) return false;
  if (((uintptr_t)a.x & 15) || ((uintptr_t)a.w & 15) || ((uintptr_t)a.y & 7)) return false;
  if (a.out_xb && ((uintptr_t)a.out_xb & 3)) return false;
  return true;
}
int gemm_small_norm_partials(const GemmArgs& a) { return a.N / 16; }

template <int E_, int NT, int MT>
static void (*small_kernel_for_c(int c))(SmallParams) {
  switch (c) {
    case 1: return gemm_small_kernel<E_, 1, NT, MT>;
    case 2: return gemm_small_kernel<E_, 2, NT, MT>;
    case 3: return gemm_small_kernel<E_, 3, NT, MT>;
    case 4: return gemm_small_kernel<E_, 4, NT, MT>;
    case 6: return gemm_small_kernel<E_, 6, NT, MT>;
    case 8: return gemm_small_kernel<E_, 8, NT, MT>;
    default: return gemm_small_kernel<E_, 12, NT, MT>;
  }
}
template <int E_, int MT>
static void (*small_kernel_for(int c, int nt))(SmallParams) {
  return nt == 1 ? small_kernel_for_c<E_, 1, MT>(c) : small_kernel_for_c<E_, 2, MT>(c);
}
// 32 weight rows per CTA when 16-row CTAs would not fit in one wave at two CTAs per SM (gate/up)
static int small_mt(const GemmArgs& a) { return a.epi == EPI_SILU_MUL && a.N % 32 == 0 && a.N / 16 > 2 * 148 ? 2 : 1; }

int gemm_small(const GemmArgs& a, cudaStream_t st) {
  if (!gemm_small_ok(a)) return SB_EUNSUPPORTED;
  SmallParams p;
  p.x = (const __nv_bfloat16*)a.x;
  p.w = (const __nv_bfloat16*)a.w;
  p.y = a.y;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.ldx = a.ldx;
  p.ns_part = a.ns_part;
  p.ns_P = a.ns_P;
  p.ns_stride = a.ns_stride;
  p.ns_eps = a.ns_eps;
  p.ns_inv_h = a.ns_inv_h;
  p.out_part = a.out_part;
  p.out_xb = (__nv_bfloat16*)a.out_xb;
  p.out_gain = (const __nv_bfloat16*)a.out_gain;
  p.trace = g_cta_trace;
  p.trace_id = g_cta_trace ? g_cta_trace_seq++ : 0;
  const int c = a.K / 256, nt = a.M <= 8 ? 1 : 2, mt = small_mt(a);
  void (*k)(SmallParams) = a.epi == EPI_STORE      ? small_kernel_for<EPI_STORE, 1>(c, nt)
                           : a.epi == EPI_RESID_ADD ? small_kernel_for<EPI_RESID_ADD, 1>(c, nt)
                           : mt == 2                ? small_kernel_for<EPI_SILU_MUL, 2>(c, nt)
                                                    : small_kernel_for<EPI_SILU_MUL, 1>(c, nt);
  return launch_k(k, dim3(a.N / (16 * mt)), dim3(SG_W * 32), 0, st, p);
}

}  // namespace sb
