// tcgen05 / TMEM / TMA GEMM for the bf16 verify forward and draft step (K2).
//
//   Y[M, N] = X[M, K] . W[N, K]^T      (bf16 in, fp32 accumulate in TMEM)
//
// Decode-shaped problems have few tokens (M = b(k+1) = 2..72 at b <= 8) and
// wide weights, so the kernel is written swap-AB: the weight tile is the MMA
// A operand (128 weight rows = UMMA_M 128), the token tile is the B operand
// (UMMA_N = M rounded up to 16, <= 256), and the accumulator D[128 x TN] lives
// in TMEM (lane = weight row, column = token).  The weight stream is the
// roofline term, so narrow matrices are split along K across a thread-block
// CLUSTER of up to 8 CTAs (enough CTAs that every SM streams, at most one
// resident wave); the cluster reduces its fp32 partial tiles through
// distributed shared memory in rank order (deterministic, no global scratch,
// no serial fixup).  Launched with programmatic dependent launch: the
// producer requests its first ring of WEIGHT tiles before griddepcontrol.wait,
// so a GEMM's weight stream overlaps the tail of the kernel that produces its
// activations.
//
// Warp roles (192 threads): warp 0 = TMA producer (one elected lane),
// warp 1 = TMEM allocator + MMA issuer (one elected lane), warps 2..5 =
// epilogue (tcgen05.ld 32x32b: warp w owns TMEM lanes 32*(w%4)..+31).
// Operands are staged by TMA with 128B swizzle into a multi-stage mbarrier
// ring; tcgen05.commit releases a stage back to the producer.
#include <cuda.h>

#include <climits>
#include <cstdio>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace sb {

constexpr int TC_THREADS = 192;
constexpr int TC_MAX_TN = 256;


struct TcParams {
  int w_hint;  // L2 policy of the weight stream: 0 default, 1 evict-first, 2 evict-last
  int k_rot;      // rotate each CTA's k-block order by tile (spreads the shared token-tile reads over L2)
  int m_fast;     // raster: 1 = the m-tiles of one weight tile are adjacent CTAs (grid.x), 0 = grid.y
  int m_tiles;
  int M, N, K;
  int tn;         // UMMA_N (tokens per tile)
  int n_tiles_n;  // ceil(N / 128)
  int kb;         // 64-wide k-blocks of K
  int splits;     // K splits == cluster size (1..8)
  int wt;         // 128-row weight tiles per CTA sharing each token (X) stage: 1, or 2 (splits == 1, large T)
  int stages;
  int epi;
  void* y;
  float* aux_val;  // EPI_ARGMAX partials [n_tiles_n][M]
  int* aux_idx;
  // fused RMSNorm, consumer side: scale token m by
  //   rsqrt(sum_p ns_part[p * ns_stride + m * ns_row_step + ns_row_off] * ns_inv_h + ns_eps)
  const float* ns_part;
  int ns_P, ns_stride, ns_row_step, ns_row_off;
  float ns_eps, ns_inv_h;
  // fused RMSNorm, producer side (EPI_RESID_ADD): xb = bf16(new residual) [M, N];
  // out_part[(tile_n * splits + split) * M + m] = sum over this CTA's rows of new^2
  float* out_part;
  __nv_bfloat16* out_xb;
  const __nv_bfloat16* out_gain;  // RMSNorm gain of the CONSUMER of xb: xb = bf16(new * gain[n]) (NULL = 1)
  const __nv_bfloat16* bias;  // OPT: per-row bias [N] added before the epilogue op
  int relu;
  unsigned long long* trace;  // sb_debug_cta_trace (NULL = off)
  int trace_id;
  int pre_max;      // ring stages of weights requested before the PDL wait (0 = all)
  int launch_late;  // 1: trigger dependents at the end of the epilogue instead of after the last load
  int dbg;          // experiments (sb_debug_gemm_pdl): bit 0 skip the epilogue stores, bit 3 plain stores,
                    // bit 4 scalar (per-element) epilogue, bit 2 the 4-8 byte row emit of store / silu tiles
  const float* ln_s1;  // fused LayerNorm (GemmArgs::ln_*, out_part1)
  const float* ln_c1;
  const float* ln_c2;
  float* out_part1;
  int vec;          // row epilogue (N % 16 == 0, 16-byte aligned outputs, power-of-two splits)
  int res_bytes;    // EPI_RESID_ADD: bytes of residual rows prefetched into shared memory (0 = loaded per row)
};

// Shared-memory scratch of the epilogue (reuses the drained operand ring).  Row epilogue: staging
// (split-K: the partial tile [tn][128] f32 the cluster reads; else [2][TC_EPI_CH][128] f32).
constexpr int TC_EPI_CH = 32;  // tokens per staged epilogue chunk (splits == 1)
__host__ __device__ inline uint32_t tc_stage_bytes(int tn, int splits) {
  return splits > 1 ? (uint32_t)tn * TC_BM * 4 : 2u * TC_EPI_CH * TC_BM * 4;
}
__host__ __device__ inline uint32_t tc_scratch_bytes(int tn, int splits, int vec, int rows_max) {
  if (vec) return tc_stage_bytes(tn, splits);
  return splits > 1 ? (uint32_t)tn * (TC_BM + rows_max) * 4 : (uint32_t)tn * 12 * 4;
}
// The prefetched residual rows live AFTER max(ring, scratch): they land while the ring is in use.
__host__ __device__ inline uint32_t tc_res_offset(uint32_t ring_bytes, uint32_t scratch_bytes) {
  return ((ring_bytes > scratch_bytes ? ring_bytes : scratch_bytes) + 127) & ~127u;
}

// (approximate division: the IEEE one costs a slow-path check + convergence barrier per element in the
// row epilogue; the product is rounded to bf16)
__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.f + __expf(-g)); }

// Epilogue stores are streaming (st.global.cs): with the weight stream saturating HBM, default
// write-back stores took ~2 us per 16-token chunk (measured: scripts/epi_micro.py, 2.40 -> 0.90 us at
// 9 tokens, 10.6 -> 3.4 us at 72); dbg bit 3 restores plain stores for A/B.
template <typename T>
__device__ __forceinline__ void st_o(const TcParams& p, T* dst, T v) {
  if (p.dbg & 8) *dst = v;
  else __stcs(dst, v);
}


// Output of one (token m, weight row n) element.  Returns the value the
// element ends with (the new residual for EPI_RESID_ADD) for norm partials.
template <int E_>
__device__ __forceinline__ float epi_one(const TcParams& p, int m, int n, float v) {
  if (m >= p.M || n >= p.N) return 0.f;
  size_t o = (size_t)m * p.N + n;
  if (p.bias) v += __bfloat162float(p.bias[n]);
  if (p.relu && E_ != EPI_RESID_ADD) v = fmaxf(v, 0.f);
  if (E_ == EPI_STORE) {
    st_o(p, (__nv_bfloat16*)p.y + o, __float2bfloat16_rn(v));
  } else if (E_ == EPI_STORE_F32) {
    st_o(p, (float*)p.y + o, v);
  } else {
    float nv = ((float*)p.y)[o] + v;
    st_o(p, (float*)p.y + o, nv);
    if (p.out_xb) st_o(p, p.out_xb + o, __float2bfloat16_rn(p.out_gain ? nv * __bfloat162float(p.out_gain[n]) : nv));
    return nv;
  }
  return v;
}
// EPI_RESID_ADD with the old residual already loaded (`prev`): lets callers
// issue all residual loads of a chunk before any store (one L2 round trip per
// chunk instead of one per element).
template <int E_>
__device__ __forceinline__ float epi_resid_pre(const TcParams& p, int m, int n, float v, float prev) {
  if (m >= p.M || n >= p.N) return 0.f;
  const size_t o = (size_t)m * p.N + n;
  if (p.bias) v += __bfloat162float(p.bias[n]);
  const float nv = prev + v;
  st_o(p, (float*)p.y + o, nv);
  if (p.out_xb) st_o(p, p.out_xb + o, __float2bfloat16_rn(p.out_gain ? nv * __bfloat162float(p.out_gain[n]) : nv));
  return nv;
}
__device__ __forceinline__ float resid_load(const TcParams& p, int m, int n) {
  return (m < p.M && n < p.N) ? __ldcg((const float*)p.y + (size_t)m * p.N + n) : 0.f;
}
// SILU pairs rows (n, n+1) = (gate, up)
__device__ __forceinline__ void epi_pair(const TcParams& p, int m, int n, float g, float u) {
  if (m >= p.M || n >= p.N) return;
  st_o(p, (__nv_bfloat16*)p.y + (size_t)m * (p.N / 2) + n / 2, __float2bfloat16_rn(silu_f(g) * u));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
}
// Row epilogue: emit token j's row of the 128-row tile at n0a (lane l holds rows 4l..4l+3 in x): the
// output op, one 8-16 byte streaming store per lane and output tensor (a warp covers the token's 128
// contiguous rows), then the norm partial / argmax of the row reduced over the warp (fixed xor trees).
// (Measured alternatives, slower in the forward: per-element stores -- one 2-4 byte store per row and
// token, ~2 us per 16 tokens under the weight stream; bulk (TMA engine) copies of rows formatted in
// shared memory -- 3.15 vs 3.01 ms verify at b=8, k=3.)
// Per-row constants of the row epilogue (lane l: rows n..n+3), loaded once per tile instead of once
// per token: a load after the previous token's stores could not be hoisted above them.
struct EmitRow {
  float4 c1, c2, bias, gain;
};
__device__ __forceinline__ float4 bf16x4_to_f4(uint2 v) {
  return make_float4(__bfloat162float(__ushort_as_bfloat16((unsigned short)(v.x & 0xffff))),
                     __bfloat162float(__ushort_as_bfloat16((unsigned short)(v.x >> 16))),
                     __bfloat162float(__ushort_as_bfloat16((unsigned short)(v.y & 0xffff))),
                     __bfloat162float(__ushort_as_bfloat16((unsigned short)(v.y >> 16))));
}
__device__ __forceinline__ EmitRow load_emit_row(const TcParams& p, int n0a, int lane) {
  const int n = n0a + 4 * lane;
  EmitRow r;
  r.c1 = r.c2 = r.bias = make_float4(0.f, 0.f, 0.f, 0.f);
  r.gain = make_float4(1.f, 1.f, 1.f, 1.f);
  if (n < p.N) {
    if (p.ln_c1) {
      r.c1 = *reinterpret_cast<const float4*>(p.ln_c1 + n);
      r.c2 = *reinterpret_cast<const float4*>(p.ln_c2 + n);
    }
    if (p.bias) r.bias = bf16x4_to_f4(*reinterpret_cast<const uint2*>(p.bias + n));
    if (p.out_gain) r.gain = bf16x4_to_f4(*reinterpret_cast<const uint2*>(p.out_gain + n));
  }
  return r;
}
template <int E_>
__device__ __forceinline__ void tc_emit_row(const TcParams& p, const EmitRow& er, int lane, int j, int jr, int acc,
                                            int tn, int m0, int n0a, int tile_a, float (&x)[4], float sc,
                                            uint64_t* res_bar, const float* rb, bool has_pre = false,
                                            float4 pre = make_float4(0.f, 0.f, 0.f, 0.f), float musc = 0.f) {
  const int m = m0 + j;
  if (m >= p.M) return;  // (warp-uniform) padding token
  const int n = n0a + 4 * lane;
  const bool nv = n < p.N;
  const size_t o = (size_t)m * p.N + n;
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] *= sc;
  if (p.ln_c1) {  // fused LayerNorm: - mean * rstd * (W gamma) + W beta
    x[0] += er.c2.x - musc * er.c1.x;
    x[1] += er.c2.y - musc * er.c1.y;
    x[2] += er.c2.z - musc * er.c1.z;
    x[3] += er.c2.w - musc * er.c1.w;
  }
  if (p.bias) {
    x[0] += er.bias.x;
    x[1] += er.bias.y;
    x[2] += er.bias.z;
    x[3] += er.bias.w;
  }
  if (E_ != EPI_RESID_ADD && p.relu)
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = fmaxf(x[i], 0.f);
  if (E_ == EPI_STORE) {
    if (nv) __stcs(reinterpret_cast<uint2*>((__nv_bfloat16*)p.y + o), make_uint2(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3])));
  } else if (E_ == EPI_STORE_F32) {
    if (nv) __stcs(reinterpret_cast<float4*>((float*)p.y + o), make_float4(x[0], x[1], x[2], x[3]));
  } else if (E_ == EPI_SILU_MUL) {
    if (nv)
      __stcs(reinterpret_cast<unsigned int*>((__nv_bfloat16*)p.y + (size_t)m * (p.N / 2) + n / 2),
             pack_bf16x2(silu_f(x[0]) * x[1], silu_f(x[2]) * x[3]));
  } else if (E_ == EPI_ARGMAX) {
    if (p.y && nv) __stcs(reinterpret_cast<float4*>((float*)p.y + o), make_float4(x[0], x[1], x[2], x[3]));
    ArgMax am{-INFINITY, INT_MAX};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (n + i < p.N && x[i] > am.v) am = ArgMax{x[i], n + i};
    am = warp_argmax(am);
    if (lane == 0 && tile_a < p.n_tiles_n) {
      st_o(p, p.aux_val + (size_t)tile_a * p.M + m, am.v);
      st_o(p, p.aux_idx + (size_t)tile_a * p.M + m, am.i);
    }
  } else {  // EPI_RESID_ADD: new residual, its bf16 copy scaled by the consumer's gain, norm partial
    float4 pr = make_float4(0.f, 0.f, 0.f, 0.f);
    if (has_pre) {  // loaded by the caller with the rest of its batch
      pr = pre;
    } else if (p.res_bytes) {
      mbar_wait(res_bar, 0);
      pr = *reinterpret_cast<const float4*>(rb + ((size_t)acc * tn + jr) * TC_BM + 4 * lane);
    } else if (nv) {
      pr = __ldcg(reinterpret_cast<const float4*>((const float*)p.y + o));
    }
    const float a0 = pr.x + x[0], a1 = pr.y + x[1], a2 = pr.z + x[2], a3 = pr.w + x[3];
    if (nv) __stcs(reinterpret_cast<float4*>((float*)p.y + o), make_float4(a0, a1, a2, a3));
    if (p.out_xb && nv) {
      const float g[4] = {er.gain.x, er.gain.y, er.gain.z, er.gain.w};
      __stcs(reinterpret_cast<uint2*>(p.out_xb + o), make_uint2(pack_bf16x2(a0 * g[0], a1 * g[1]), pack_bf16x2(a2 * g[2], a3 * g[3])));
    }
    if (p.out_part) {
      const float sq = warp_sum(nv ? ((a0 * a0 + a1 * a1) + a2 * a2) + a3 * a3 : 0.f);
      if (lane == 0 && tile_a < p.n_tiles_n) st_o(p, p.out_part + (size_t)tile_a * p.M + m, sq);
    }
    if (p.out_part1) {  // (LayerNorm consumers also need the sum)
      const float s1 = warp_sum(nv ? ((a0 + a1) + a2) + a3 : 0.f);
      if (lane == 0 && tile_a < p.n_tiles_n) st_o(p, p.out_part1 + (size_t)tile_a * p.M + m, s1);
    }
  }
}

// Rows of the 128-row tile reduced by cluster rank `split` (pairs, so the
// silu(gate)*up epilogue never straddles two ranks): [2*(split*64/s), 2*((split+1)*64/s)).
__host__ __device__ __forceinline__ int split_row_lo(int split, int splits) { return 2 * (split * (TC_BM / 2) / splits); }
__host__ __device__ __forceinline__ int split_rows_max(int splits) { return 2 * ((TC_BM / 2 + splits - 1) / splits); }

// grid = (n_tiles_n * splits, m_tiles), cluster = (splits, 1, 1): the `splits`
// CTAs of a cluster share one 128 x tn output tile and split its K range.
template <int E_, int V_>
__global__ void __launch_bounds__(TC_THREADS, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ unsigned long long tr_t[5];
  if (p.trace && threadIdx.x == 0) tr_t[4] = 0;
  if (p.trace && threadIdx.x == 0) tr_t[0] = gtime();
  // 1024-aligned base by pointer arithmetic on smem_raw (keeps the shared address space visible to the
  // compiler: STS / LDS instead of generic ST / LD for the epilogue staging)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tn = p.tn;
  const int wt = p.wt;
  const uint32_t a_bytes = wt * TC_BM * TC_BK * 2;
  const uint32_t b_bytes = tn * TC_BK * 2;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  const uint32_t ring_bytes = p.stages * stage_bytes;
  // scratch (reuses the drained ring): split>1: partial tile [tn][128] + squares [tn][rows_max];
  // split==1: argmax staging [2][4][tn] + squares [4][tn]
  const uint32_t scratch_bytes = tc_scratch_bytes(tn, p.splits, V_, split_rows_max(p.splits));
  uint8_t* stage_base = smem;
  float* res_rows = (float*)(smem + tc_res_offset(ring_bytes, scratch_bytes));  // [wt][tn][128] (res_bytes)
  uint64_t* full = (uint64_t*)(smem + tc_res_offset(ring_bytes, scratch_bytes) + p.res_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* tmem_full = empty + p.stages;
  uint64_t* res_bar = tmem_full + 1;  // prefetched residual rows landed (row epilogue)
  uint32_t* tmem_slot = (uint32_t*)(res_bar + 1);
  float* inv_s = (float*)(tmem_slot + 4);  // [tn] per-token 1/rms (fused RMSNorm) / rstd (fused LayerNorm)
  float* nsum = inv_s + tn;                 // [4][tn] per-token partial sums of squares (fused RMSNorm)
  float* musc = nsum + 4 * tn;              // [tn] fused LayerNorm: mean * rstd
  float* nsum1 = musc + tn;                 // [4][tn] fused LayerNorm: partial sums of x
  float* red = (float*)smem;               // split-K partial tile [tn][128] (reuses the drained ring)
  float* sq = p.splits > 1 ? red + tn * TC_BM : red + 8 * tn;  // norm squares staging

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = p.splits > 1 ? (int)cluster_rank() : 0;
  // m-fast raster: the token tiles sharing a weight tile run in the same wave,
  // so the weight tile streams from HBM once and the others hit L2
  const int mn = blockIdx.x / p.splits;
  const int tile_n = p.m_fast ? mn / p.m_tiles : mn;  // in units of wt 128-row tiles
  const int n0 = tile_n * TC_BM * wt;
  const int m0 = (p.m_fast ? mn % p.m_tiles : (int)blockIdx.y) * tn;
  const int kb0 = (int)((long long)split * p.kb / p.splits);
  const int kb1 = (int)((long long)(split + 1) * p.kb / p.splits);
  const int nkb = kb1 - kb0;
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < wt * tn) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(res_bar, 1);
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

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer.  Weights never depend on the previous
      // kernel, so the first ring of weight tiles is requested BEFORE the
      // programmatic-dependency wait: under PDL the weight stream of this GEMM
      // overlaps the tail of the kernel that produces its activations.
      int pre = nkb < p.stages ? nkb : p.stages;
      if (p.pre_max > 0 && pre > p.pre_max) pre = p.pre_max;
      // single token tile (decode): every CTA reads the same X k-block at the same time -> rotate
      // each weight tile's k order to spread those reads over L2 (several token tiles share the
      // weight tile instead: keep their k order aligned so the weight stream hits L2)
      const int rot = (p.k_rot && p.m_tiles == 1) ? (int)((tile_n * 7u) % (unsigned)nkb) : 0;
      const uint64_t wpol = p.w_hint == 2 ? l2_policy_evict_last() : l2_policy_evict_first();
      auto kb_of = [&](int i) { const int j = i + rot; return kb0 + (j >= nkb ? j - nkb : j); };
      if (p.dbg & 64) griddep_launch();  // experiment: dependents may launch right away
      for (int i = 0; i < pre; ++i) {
        uint8_t* sa = stage_base + i * stage_bytes;
        mbar_expect_tx(&full[i], stage_bytes);
        if (p.w_hint) tma_load_2d_hint(sa, &map_w, &full[i], kb_of(i) * TC_BK, n0, wpol);
        else tma_load_2d(sa, &map_w, &full[i], kb_of(i) * TC_BK, n0);
      }
      griddep_wait();
      if (p.trace) tr_t[1] = gtime();
      for (int i = 0; i < pre; ++i)
        tma_load_2d(stage_base + i * stage_bytes + a_bytes, &map_x, &full[i], kb_of(i) * TC_BK, m0);
      int stage = pre % p.stages;
      uint32_t phase = (pre == p.stages) ? 1u : 0u;
      for (int i = pre; i < nkb; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = stage_base + stage * stage_bytes;
        mbar_expect_tx(&full[stage], stage_bytes);
        if (p.w_hint) tma_load_2d_hint(sa, &map_w, &full[stage], kb_of(i) * TC_BK, n0, wpol);
        else tma_load_2d(sa, &map_w, &full[stage], kb_of(i) * TC_BK, n0);
        tma_load_2d(sa + a_bytes, &map_x, &full[stage], kb_of(i) * TC_BK, m0);
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (!p.launch_late) griddep_launch();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread)
      const uint32_t idesc = make_idesc(tn);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nkb; ++i) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (p.trace && i == 0) tr_t[2] = gtime();
        uint32_t sa = smem_u32(stage_base + stage * stage_bytes);
        uint32_t sb = sa + a_bytes;
        for (int a = 0; a < wt; ++a) {  // the X stage feeds every weight tile of the CTA
#pragma unroll
          for (int kk = 0; kk < TC_BK / TC_UK; ++kk)
            tc_mma(tmem + (uint32_t)(a * tn), sw128_desc(sa + a * TC_BM * TC_BK * 2 + kk * TC_UK * 2),
                   sw128_desc(sb + kk * TC_UK * 2), idesc, (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(&empty[stage]);
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      tc_commit(tmem_full);
    }
  } else {
    // ---------------- epilogue warps: TMEM -> registers -> (DSMEM reduce) -> global
    griddep_wait();
    const int et = threadIdx.x - 64;
    if (V_ && p.res_bytes && et == 0) {
      // the residual rows this CTA will update (final since the previous kernel completed) head for
      // shared memory now, under the weight stream: one 512-byte bulk copy per (tile, token)
      const int jlo = p.splits > 1 ? split * tn / p.splits : 0, jhi = p.splits > 1 ? (split + 1) * tn / p.splits : tn;
      const int nj = min(jhi, p.M - m0) - jlo;
      float* rb = res_rows;
      if (nj > 0) {
        int nt = 0;
        for (int a = 0; a < wt; ++a) nt += (n0 + a * TC_BM < p.N) ? 1 : 0;
        mbar_expect_tx(res_bar, (uint32_t)(nt * nj * TC_BM * 4));
        for (int a = 0; a < nt; ++a)
          for (int j = 0; j < nj; ++j)
            bulk_g2s_bar(rb + ((size_t)a * tn + j) * TC_BM, (const float*)p.y + (size_t)(m0 + jlo + j) * p.N + n0 + a * TC_BM,
                         TC_BM * 4, res_bar);
      } else {
        mbar_arrive(res_bar);
      }
    }
    const int quad = warp & 3;
    const int row = quad * 32 + lane;  // weight row within the tile (= TMEM lane)
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    // fused RMSNorm (consumer): per-token 1/rms from the producer's partials,
    // computed while the weights stream (these warps are otherwise idle)
    if (p.ns_part) {
      // the producer GEMM left ns_P partial sums of squares per token (one per
      // 128-row tile and split): 4 fixed sub-ranges per token, each summed 8
      // loads at a time by one thread, combined in order -- deterministic and
      // independent of the token count (batch invariance); the loads overlap
      // the weight stream of this GEMM
      constexpr int tpj = 4;
      for (int jj = et; jj < tn * tpj; jj += 128) {
        const int j = jj % tn, part = jj / tn;
        const int m = m0 + j;
        const int q0 = part * p.ns_P / tpj, q1 = (part + 1) * p.ns_P / tpj;
        float acc = 0.f;
        if (m < p.M) {
          const float* src = p.ns_part + (size_t)m * p.ns_row_step + p.ns_row_off;
          for (int q = q0; q < q1; q += 8) {
            float t8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) t8[i] = q + i < q1 ? __ldcg(src + (size_t)(q + i) * p.ns_stride) : 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) acc += t8[i];
          }
        }
        nsum[part * tn + j] = acc;
        if (p.ln_s1) {  // fused LayerNorm: the sums of x the same way
          float a1 = 0.f;
          if (m < p.M) {
            const float* src = p.ln_s1 + (size_t)m * p.ns_row_step + p.ns_row_off;
            for (int q = q0; q < q1; q += 8) {
              float t8[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) t8[i] = q + i < q1 ? __ldcg(src + (size_t)(q + i) * p.ns_stride) : 0.f;
#pragma unroll
              for (int i = 0; i < 8; ++i) a1 += t8[i];
            }
          }
          nsum1[part * tn + j] = a1;
        }
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      for (int j = et; j < tn; j += 128) {
        float tot = nsum[j];
        for (int part = 1; part < tpj; ++part) tot += nsum[part * tn + j];
        if (p.ln_s1) {  // LayerNorm: mean = S1 / H, var = S2 / H - mean^2, rstd = rsqrt(var + eps)
          float t1 = nsum1[j];
          for (int part = 1; part < tpj; ++part) t1 += nsum1[part * tn + j];
          const float mean = t1 * p.ns_inv_h;
          const float var = fmaxf(tot * p.ns_inv_h - mean * mean, 0.f);
          const float rstd = rsqrtf(var + p.ns_eps);
          inv_s[j] = rstd;
          musc[j] = mean * rstd;
        } else {
          inv_s[j] = rsqrtf(tot * p.ns_inv_h + p.ns_eps);
        }
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
    }
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    if (p.trace && et == 0) tr_t[3] = gtime();
    const bool scale = p.ns_part != nullptr;
    if (V_) {
      if (p.splits > 1) {
        // split-K: dump this CTA's partial tile for the cluster (reduced after the cluster barrier)
        for (int j0 = 0; j0 < tn; j0 += 16) {
          float v[16];
          tmem_ld16(lane_addr + (uint32_t)j0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) red[(j0 + j) * TC_BM + row] = v[j];
        }
      } else {
        // Each chunk of up to 32 tokens goes TMEM -> registers -> shared memory ([32][128] f32,
        // double-buffered; one tcgen05.wait per chunk), then warp ew emits tokens ew, ew+4, ...:
        // lane l owns rows 4l..4l+3 of the token's row.
        const int ew = warp - 2;
        int ci = 0;
        for (int acc = 0; acc < wt; ++acc) {
          const EmitRow er = load_emit_row(p, n0 + acc * TC_BM, lane);
          for (int j0 = 0; j0 < tn; j0 += TC_EPI_CH, ++ci) {
            float* sb = red + (ci & 1) * TC_EPI_CH * TC_BM;
            const int cn = min(TC_EPI_CH, tn - j0);  // 16 or 32 (tn % 16 == 0)
            {
              uint32_t r0[16], r1[16];
              tmem_ld16_nw(lane_addr + (uint32_t)(acc * tn) + j0, r0);
              if (cn > 16) tmem_ld16_nw(lane_addr + (uint32_t)(acc * tn) + j0 + 16, r1);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 16; ++j) sb[j * TC_BM + row] = __uint_as_float(r0[j]);
              if (cn > 16)
#pragma unroll
                for (int j = 0; j < 16; ++j) sb[(16 + j) * TC_BM + row] = __uint_as_float(r1[j]);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (p.trace && et == 0 && ci == 0) tr_t[4] = gtime();
            if (p.dbg & 2) continue;  // experiment: TMEM -> shared staging only, no emit
            if (E_ == EPI_STORE && !(p.dbg & 4) && !p.bias && !p.relu && !p.ln_c1) {
              // wide emit: lane (h, q) takes rows 8q..8q+7 of token 2*ew + h (+8 ...): one 16-byte store;
              // a warp instruction covers 2 tokens
              const int h = lane >> 4, q = lane & 15;
              const int nq0 = n0 + acc * TC_BM + 8 * q;
              for (int jb = 2 * ew + h; jb < cn; jb += 8) {
                const int j = j0 + jb, m = m0 + j;
                const float4 v0 = *reinterpret_cast<const float4*>(sb + jb * TC_BM + 8 * q);
                const float4 v1 = *reinterpret_cast<const float4*>(sb + jb * TC_BM + 8 * q + 4);
                const float sc = scale ? inv_s[j] : 1.f;
                if (m < p.M && nq0 < p.N)
                  __stcs(reinterpret_cast<uint4*>((__nv_bfloat16*)p.y + (size_t)m * p.N + nq0),
                         make_uint4(pack_bf16x2(v0.x * sc, v0.y * sc), pack_bf16x2(v0.z * sc, v0.w * sc),
                                    pack_bf16x2(v1.x * sc, v1.y * sc), pack_bf16x2(v1.z * sc, v1.w * sc)));
              }
              continue;
            }
            if (E_ == EPI_RESID_ADD && !(p.dbg & 4) && !p.bias && !p.relu && !p.ln_c1 && !p.out_part1) {
              // wide emit: lane (h, q) updates rows 8q..8q+7 of token 2*ew + h (+8 ...): two 16-byte fp32
              // residual stores and one 16-byte bf16*gain store; the token's norm partial is summed over
              // the 16 lanes of its half-warp (fixed xor tree)
              const int h = lane >> 4, q = lane & 15;
              const int n = n0 + acc * TC_BM + 8 * q;
              const bool nv = n < p.N;
              float gn[8] = {1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f};
              if (p.out_gain && nv) {
                const uint4 g4 = *reinterpret_cast<const uint4*>(p.out_gain + n);
                const float4 ga = bf16x4_to_f4(make_uint2(g4.x, g4.y)), gb = bf16x4_to_f4(make_uint2(g4.z, g4.w));
                gn[0] = ga.x, gn[1] = ga.y, gn[2] = ga.z, gn[3] = ga.w, gn[4] = gb.x, gn[5] = gb.y, gn[6] = gb.z, gn[7] = gb.w;
              }
              if (p.res_bytes) mbar_wait(res_bar, 0);
              // all residual rows of the lane's (<= 4) tokens in flight before the first store
              constexpr int NI = TC_EPI_CH / 8;
              float4 rw[NI][2];
#pragma unroll
              for (int i = 0; i < NI; ++i) {
                const int jb = 2 * ew + h + 8 * i, j = j0 + jb, m = m0 + j;
                rw[i][0] = rw[i][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (jb >= cn) continue;
                if (p.res_bytes) {
                  const float* rr = res_rows + ((size_t)acc * tn + j) * TC_BM + 8 * q;
                  rw[i][0] = *reinterpret_cast<const float4*>(rr);
                  rw[i][1] = *reinterpret_cast<const float4*>(rr + 4);
                } else if (m < p.M && nv) {
                  const float* rr = (const float*)p.y + (size_t)m * p.N + n;
                  rw[i][0] = __ldcg(reinterpret_cast<const float4*>(rr));
                  rw[i][1] = __ldcg(reinterpret_cast<const float4*>(rr + 4));
                }
              }
#pragma unroll
              for (int i = 0; i < NI; ++i) {
                const int jb = 2 * ew + h + 8 * i;
                if (jb >= cn) break;  // (uniform across the warp's halves: cn is a multiple of 16)
                const int j = j0 + jb, m = m0 + j;
                const bool ok = m < p.M && nv;
                const float4 v0 = *reinterpret_cast<const float4*>(sb + jb * TC_BM + 8 * q);
                const float4 v1 = *reinterpret_cast<const float4*>(sb + jb * TC_BM + 8 * q + 4);
                const float4 r0 = rw[i][0], r1 = rw[i][1];
                const float sc = scale ? inv_s[j] : 1.f;
                const float a[8] = {r0.x + v0.x * sc, r0.y + v0.y * sc, r0.z + v0.z * sc, r0.w + v0.w * sc,
                                    r1.x + v1.x * sc, r1.y + v1.y * sc, r1.z + v1.z * sc, r1.w + v1.w * sc};
                if (ok) {
                  float* yo = (float*)p.y + (size_t)m * p.N + n;
                  __stcs(reinterpret_cast<float4*>(yo), make_float4(a[0], a[1], a[2], a[3]));
                  __stcs(reinterpret_cast<float4*>(yo + 4), make_float4(a[4], a[5], a[6], a[7]));
                  if (p.out_xb)
                    __stcs(reinterpret_cast<uint4*>(p.out_xb + (size_t)m * p.N + n),
                           make_uint4(pack_bf16x2(a[0] * gn[0], a[1] * gn[1]), pack_bf16x2(a[2] * gn[2], a[3] * gn[3]),
                                      pack_bf16x2(a[4] * gn[4], a[5] * gn[5]), pack_bf16x2(a[6] * gn[6], a[7] * gn[7])));
                }
                if (p.out_part) {
                  float sq = ok ? (((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]) + a[3] * a[3]) +
                                      (((a[4] * a[4] + a[5] * a[5]) + a[6] * a[6]) + a[7] * a[7])
                                : 0.f;
#pragma unroll
                  for (int o = 1; o < 16; o <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
                  const int ta = tile_n * wt + acc;
                  if (q == 0 && m < p.M && ta < p.n_tiles_n) st_o(p, p.out_part + (size_t)ta * p.M + m, sq);
                }
              }
              continue;
            }
            if (E_ == EPI_SILU_MUL && !(p.dbg & 4) && !p.bias && !p.relu && !p.ln_c1) {
              // wide emit: lane (sub, q) takes 16 rows of token 4*ew + sub (+16 ...): 8 silu outputs, one
              // 16-byte store; a warp instruction covers 4 tokens.  Under the weight stream of the other
              // CTAs the emit is bound by store instructions, not bytes: silu epilogue 3.4 -> 2.0 us at
              // 64 tokens, 24 -> 13 us at 1016 (scripts/epi_wide.py; outputs bit-identical)
              const int sub = lane >> 3, q = lane & 7;
              const int nq0 = n0 + acc * TC_BM + 16 * q;
              for (int jb = 4 * ew + sub; jb < cn; jb += 16) {
                const int j = j0 + jb, m = m0 + j;
                const float* src = sb + jb * TC_BM + 16 * q;
                float f[16];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const float4 v4 = *reinterpret_cast<const float4*>(src + 4 * c);
                  f[4 * c + 0] = v4.x;
                  f[4 * c + 1] = v4.y;
                  f[4 * c + 2] = v4.z;
                  f[4 * c + 3] = v4.w;
                }
                const float sc = scale ? inv_s[j] : 1.f;
                uint32_t o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float g0 = f[4 * i] * sc, u0 = f[4 * i + 1] * sc, g1 = f[4 * i + 2] * sc, u1 = f[4 * i + 3] * sc;
                  o[i] = pack_bf16x2(silu_f(g0) * u0, silu_f(g1) * u1);
                }
                if (m < p.M && nq0 < p.N)
                  __stcs(reinterpret_cast<uint4*>((__nv_bfloat16*)p.y + (size_t)m * (p.N / 2) + nq0 / 2),
                         make_uint4(o[0], o[1], o[2], o[3]));
              }
              continue;
            }
            // EPI_RESID_ADD without the smem prefetch (large tiles): the warp's residual rows of the
            // chunk are loaded together (one round trip per chunk: prefill o / down epilogue 53 -> 27 us)
            // All of the warp's staged rows (and residual rows) are loaded before its first store:
            // the token emits are then independent chains the scheduler interleaves.
            constexpr bool RL = E_ == EPI_RESID_ADD;
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            float4 a8[TC_EPI_CH / 4], res8[TC_EPI_CH / 4];
            if (!RL)  // (the residual epilogue keeps its staged reads per token: register budget at 2 CTAs/SM)
#pragma unroll
              for (int i = 0; i < TC_EPI_CH / 4; ++i) {
                const int jl = ew + 4 * i;
                a8[i] = jl < cn ? *reinterpret_cast<const float4*>(sb + jl * TC_BM + 4 * lane) : z4;
              }
            if (RL) {
              const int n = n0 + acc * TC_BM + 4 * lane;
              if (p.res_bytes) mbar_wait(res_bar, 0);
#pragma unroll
              for (int i = 0; i < TC_EPI_CH / 4; ++i) {
                const int jl = ew + 4 * i;
                const int m = m0 + j0 + jl;
                if (p.res_bytes)
                  res8[i] = jl < cn ? *reinterpret_cast<const float4*>(res_rows + ((size_t)acc * tn + j0 + jl) * TC_BM + 4 * lane) : z4;
                else
                  res8[i] = (jl < cn && m < p.M && n < p.N)
                                ? __ldcg(reinterpret_cast<const float4*>((const float*)p.y + (size_t)m * p.N + n))
                                : z4;
              }
            }
#pragma unroll
            for (int i = 0; i < TC_EPI_CH / 4; ++i) {
              const int jl = ew + 4 * i;
              if (jl >= cn) break;
              const int j = j0 + jl;
              const float4 a = RL ? *reinterpret_cast<const float4*>(sb + jl * TC_BM + 4 * lane) : a8[i];
              float x[4] = {a.x, a.y, a.z, a.w};
              tc_emit_row<E_>(p, er, lane, j, j, acc, tn, m0, n0 + acc * TC_BM, tile_n * wt + acc, x,
                              scale ? inv_s[j] : 1.f, res_bar, res_rows, RL, RL ? res8[i] : z4,
                              p.ln_s1 ? musc[j] : 0.f);
            }
          }
        }
      }
    } else
    for (int acc = 0; acc < wt; ++acc) {
    const int n0a = n0 + acc * TC_BM;             // this accumulator's weight rows
    const int tile_a = tile_n * wt + acc;          // its 128-row tile index
    if (acc > 0) asm volatile("bar.sync 1, 128;" ::: "memory");  // staging reuse
    for (int j0 = 0; j0 < tn; j0 += 16) {
      float v[16];
      tmem_ld16(lane_addr + (uint32_t)(acc * tn) + j0, v);
      if (p.dbg & 1) {  // experiment: no epilogue stores
        if (v[0] == 12345.f) ((float*)p.y)[0] = v[1];
        continue;
      }
      if (p.splits > 1) {
#pragma unroll
        for (int j = 0; j < 16; ++j) red[(j0 + j) * TC_BM + row] = v[j];
        continue;
      }
      if (scale) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] *= inv_s[j0 + j];
      }
      if (E_ == EPI_ARGMAX) {
        // per token: warp argmax over its 32 rows (ties -> lowest row), staged per quadrant
        float* qv = red;
        int* qi = reinterpret_cast<int*>(red + 4 * tn);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = m0 + j0 + j, n = n0a + row;
          float val = (n < p.N) ? v[j] : -INFINITY;
          if (p.y && m < p.M && n < p.N) st_o(p, (float*)p.y + (size_t)m * p.N + n, v[j]);
          ArgMax a = warp_argmax(ArgMax{val, n < p.N ? n : INT_MAX});
          if (lane == 0) {
            qv[quad * tn + j0 + j] = a.v;
            qi[quad * tn + j0 + j] = a.i;
          }
        }
      } else if (E_ == EPI_SILU_MUL) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float other = __shfl_xor_sync(0xffffffffu, v[j], 1);
          if (!(lane & 1)) epi_pair(p, m0 + j0 + j, n0a + row, v[j], other);
        }
      } else {
        float rv[16];
        if (E_ == EPI_RESID_ADD) {
#pragma unroll
          for (int j = 0; j < 16; ++j) rv[j] = resid_load(p, m0 + j0 + j, n0a + row);  // all in flight
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float nv = E_ == EPI_RESID_ADD ? epi_resid_pre<E_>(p, m0 + j0 + j, n0a + row, v[j], rv[j])
                                            : epi_one<E_>(p, m0 + j0 + j, n0a + row, v[j]);
          if (p.out_part) {  // per-token sum of squares over the tile's 128 rows (fixed xor tree)
            float s = warp_sum(nv * nv);
            if (lane == 0) sq[quad * tn + j0 + j] = s;
          }
        }
      }
    }
    if (p.splits == 1 && (E_ == EPI_ARGMAX || p.out_part) && tile_a < p.n_tiles_n) {
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int j = et; j < tn; j += 128) {
        const int m = m0 + j;
        if (m >= p.M) continue;
        if (E_ == EPI_ARGMAX) {
          const float* qv = red;
          const int* qi = reinterpret_cast<const int*>(red + 4 * tn);
          ArgMax a{qv[j], qi[j]};
#pragma unroll
          for (int q = 1; q < 4; ++q) a = argmax_merge(a, ArgMax{qv[q * tn + j], qi[q * tn + j]});
          st_o(p, p.aux_val + (size_t)tile_a * p.M + m, a.v);
          st_o(p, p.aux_idx + (size_t)tile_a * p.M + m, a.i);
        } else {
          st_o(p, p.out_part + (size_t)tile_a * p.M + m, ((sq[j] + sq[tn + j]) + sq[2 * tn + j]) + sq[3 * tn + j]);
        }
      }
    }
    }  // acc
    tc_fence_before();
  }
  __syncwarp();
  if (p.splits > 1) {
    // deterministic split-K reduction through distributed shared memory:
    // CTA `split` owns rows [split*R, (split+1)*R) of the tile and sums the
    // cluster's partials in rank order 0..splits-1.
    cluster_sync_all();
    if (V_) {
      if (warp >= 2) {
      // rank `split` owns tokens [jlo, jhi) of the tile, all 128 rows: warp ew reduces token jlo+ew,
      // +4, ... (lane l: rows 4l..4l+3, one v4 DSMEM load per rank, summed in rank order) and emits it
      const int ew = warp - 2;
      const uint32_t red_addr = smem_u32(red);
      const bool scale = p.ns_part != nullptr;
      const int jlo = split * tn / p.splits, jhi = (split + 1) * tn / p.splits;
      const EmitRow er = load_emit_row(p, n0, lane);
      constexpr bool RL = E_ == EPI_RESID_ADD;
      for (int jb = jlo + ew; jb < jhi; jb += 16) {  // groups of 4 tokens per warp
        float4 res4[4];  // residual rows of the group (no smem prefetch: large tiles), loads in flight together
        if (RL && !p.res_bytes) {
          const int n = n0 + 4 * lane;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int m = m0 + jb + 4 * i;
            res4[i] = (jb + 4 * i < jhi && m < p.M && n < p.N)
                          ? __ldcg(reinterpret_cast<const float4*>((const float*)p.y + (size_t)m * p.N + n))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        if (E_ == EPI_STORE && !(p.dbg & 4) && !p.bias && !p.relu && !p.ln_c1 && p.splits <= 2) {
          // wide emit (as in the chunk path): lane (h, q) sums rows 8q..8q+7 of tokens jb + h, jb + 2h'...
          // over the ranks in order and emits them with one 16-byte store; the warp's 4 tokens of the
          // group are covered by 2 instructions
          const int h = lane >> 4, q = lane & 15;
          const int n = n0 + 8 * q;
          float4 tw[2][2][2];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const int j = jb + 4 * (2 * i + h);
              if (j < jhi && r < p.splits) {
                tw[i][r][0] = ld_dsmem_v4_nc(red_addr + (uint32_t)((j * TC_BM + 8 * q) * 4), r);
                tw[i][r][1] = ld_dsmem_v4_nc(red_addr + (uint32_t)((j * TC_BM + 8 * q + 4) * 4), r);
              }
            }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int j = jb + 4 * (2 * i + h);
            if (j >= jhi) continue;
            float x[8] = {tw[i][0][0].x, tw[i][0][0].y, tw[i][0][0].z, tw[i][0][0].w,
                          tw[i][0][1].x, tw[i][0][1].y, tw[i][0][1].z, tw[i][0][1].w};
            if (p.splits > 1) {
              x[0] += tw[i][1][0].x;
              x[1] += tw[i][1][0].y;
              x[2] += tw[i][1][0].z;
              x[3] += tw[i][1][0].w;
              x[4] += tw[i][1][1].x;
              x[5] += tw[i][1][1].y;
              x[6] += tw[i][1][1].z;
              x[7] += tw[i][1][1].w;
            }
            const float sc = scale ? inv_s[j] : 1.f;
            const int m = m0 + j;
            if (m < p.M && n < p.N)
              __stcs(reinterpret_cast<uint4*>((__nv_bfloat16*)p.y + (size_t)m * p.N + n),
                     make_uint4(pack_bf16x2(x[0] * sc, x[1] * sc), pack_bf16x2(x[2] * sc, x[3] * sc),
                                pack_bf16x2(x[4] * sc, x[5] * sc), pack_bf16x2(x[6] * sc, x[7] * sc)));
          }
        } else if (p.splits <= 2) {
          // two ranks: the group's 4 x 2 partial rows load together (one DSMEM round trip per group)
          float4 t2[4][2];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int j = jb + 4 * i;
              if (j < jhi && q < p.splits) t2[i][q] = ld_dsmem_v4_nc(red_addr + (uint32_t)((j * TC_BM + 4 * lane) * 4), q);
            }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int j = jb + 4 * i;
            if (j >= jhi) break;
            float x[4] = {t2[i][0].x, t2[i][0].y, t2[i][0].z, t2[i][0].w};
            if (p.splits > 1) {
              x[0] += t2[i][1].x;
              x[1] += t2[i][1].y;
              x[2] += t2[i][1].z;
              x[3] += t2[i][1].w;
            }
            tc_emit_row<E_>(p, er, lane, j, j - jlo, 0, tn, m0, n0, tile_n, x, scale ? inv_s[j] : 1.f, res_bar,
                            res_rows, RL && !p.res_bytes, res4[i], p.ln_s1 ? musc[j] : 0.f);
          }
        } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = jb + 4 * i;
          if (j >= jhi) break;
          float4 t[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < p.splits) t[q] = ld_dsmem_v4_nc(red_addr + (uint32_t)((j * TC_BM + 4 * lane) * 4), q);
          float x[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < p.splits) {
              x[0] += t[q].x;
              x[1] += t[q].y;
              x[2] += t[q].z;
              x[3] += t[q].w;
            }
          tc_emit_row<E_>(p, er, lane, j, j - jlo, 0, tn, m0, n0, tile_n, x, scale ? inv_s[j] : 1.f, res_bar, res_rows,
                          RL && !p.res_bytes, res4[i], p.ln_s1 ? musc[j] : 0.f);
        }
        }
      }
      }
    } else if (warp >= 2) {
      const int r_base = split_row_lo(split, p.splits);
      const int R = split_row_lo(split + 1, p.splits) - r_base;
      const int et = threadIdx.x - 64;
      const uint32_t red_addr = smem_u32(red);
      const bool scale = p.ns_part != nullptr;
      // Batches of 4 elements per thread: all DSMEM partial loads of the batch
      // (4 x splits) and its residual loads are in flight together; the sums
      // still run in rank order 0..splits-1 (bit-identical to one at a time).
      constexpr int EB = 4;
      if (E_ == EPI_SILU_MUL) {
        const int pairs = R / 2;
        for (int it0 = et; it0 < pairs * tn; it0 += 128 * EB) {
          float t[8][EB][2];
          int rr[EB], jj[EB];
#pragma unroll
          for (int e = 0; e < EB; ++e) {
            const int it = it0 + e * 128;
            rr[e] = it < pairs * tn ? r_base + 2 * (it % pairs) : -1;
            jj[e] = it / pairs;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int e = 0; e < EB; ++e) {
              const bool ok = q < p.splits && rr[e] >= 0;
              const uint32_t ad = red_addr + (uint32_t)((jj[e] * TC_BM + (ok ? rr[e] : 0)) * 4);
              t[q][e][0] = ok ? ld_dsmem_f32_nc(ad, q) : 0.f;
              t[q][e][1] = ok ? ld_dsmem_f32_nc(ad + 4, q) : 0.f;
            }
#pragma unroll
          for (int e = 0; e < EB; ++e) {
            if (rr[e] < 0) continue;
            float g = 0.f, u = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < p.splits) {
                g += t[q][e][0];
                u += t[q][e][1];
              }
            if (scale) {
              g *= inv_s[jj[e]];
              u *= inv_s[jj[e]];
            }
            epi_pair(p, m0 + jj[e], n0 + rr[e], g, u);
          }
        }
      } else {
        for (int it0 = et; it0 < R * tn; it0 += 128 * EB) {
          float t[8][EB], rv[EB];
          int rl_[EB], jj[EB];
#pragma unroll
          for (int e = 0; e < EB; ++e) {
            const int it = it0 + e * 128;
            rl_[e] = it < R * tn ? it % R : -1;
            jj[e] = it / R;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int e = 0; e < EB; ++e) {
              const bool ok = q < p.splits && rl_[e] >= 0;
              t[q][e] = ok ? ld_dsmem_f32_nc(red_addr + (uint32_t)((jj[e] * TC_BM + r_base + rl_[e]) * 4), q) : 0.f;
            }
          if (E_ == EPI_RESID_ADD) {
#pragma unroll
            for (int e = 0; e < EB; ++e) rv[e] = rl_[e] >= 0 ? resid_load(p, m0 + jj[e], n0 + r_base + rl_[e]) : 0.f;
          }
#pragma unroll
          for (int e = 0; e < EB; ++e) {
            if (rl_[e] < 0) continue;
            float a = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < p.splits) a += t[q][e];
            if (scale) a *= inv_s[jj[e]];
            const int r = r_base + rl_[e];
            const float nv = E_ == EPI_RESID_ADD ? epi_resid_pre<E_>(p, m0 + jj[e], n0 + r, a, rv[e])
                                                    : epi_one<E_>(p, m0 + jj[e], n0 + r, a);
            if (p.out_part) sq[jj[e] * R + rl_[e]] = nv * nv;
          }
        }
        if (p.out_part) {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          for (int j = et; j < tn; j += 128) {
            const int m = m0 + j;
            if (m >= p.M) continue;
            float s = 0.f;
            for (int rl = 0; rl < R; ++rl) s += sq[j * R + rl];
            st_o(p, p.out_part + ((size_t)tile_n * p.splits + split) * p.M + m, s);
          }
        }
      }
    }
    cluster_sync_relaxed();
  }
  tc_fence_before();
  __syncthreads();
  if (p.launch_late) griddep_launch();
  if (p.trace && threadIdx.x == 0) cta_trace_write(p.trace, p.trace_id, 1, tr_t);
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

int make_map(CUtensorMap* map, const void* base, int rows, int cols, int ld, int box_rows) {
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

int num_sms() {
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

int g_pdl = 1;  // programmatic dependent launch for every forward kernel (sb_set_pdl)
int g_gemm_pre_max = 0, g_gemm_launch_late = 0, g_gemm_dbg = 0;  // sb_debug_gemm_pdl experiments
// tuning overrides (sb_gemm_tune): 0 = automatic
static int g_tune_cps = 0, g_tune_stages = 0, g_tune_splits = 0;

struct TcPlan {
  int tn, n_tiles_n, m_tiles, kb, splits, stages, ctas_per_sm, wt;
  size_t smem;
  int vec, res_bytes;
};
struct TcTuned {
  int cps, splits, wt, tn;  // tn 0: token tile of tn_for(M)
};

// Measured (CTAs per SM, K splits) per GEMM shape (sb_gemm_autotune, run by the
// host outside graph capture for the token counts an engine will use); the
// heuristic below is the fallback.
static std::mutex g_tuned_mu;
static std::map<unsigned long long, TcTuned> g_tuned;
static int g_tune_wt = 0;  // autotune candidate override (0 = plan's choice)
static int g_tune_tn = 0;  // autotune candidate token tile (0 = tn_for(M))
int g_w_l2_hint = 0;       // set per forward: large models stream weights evict-first, small ones keep them
static unsigned long long tune_key(int tn, int m_tiles, int N, int K) {
  return ((unsigned long long)tn << 48) | ((unsigned long long)m_tiles << 40) | ((unsigned long long)N << 20) |
         (unsigned long long)K;
}

static void tc_plan_smem(TcPlan& q) {
  const size_t stage = (size_t)(TC_BM * q.wt + q.tn) * TC_BK * 2;
  const size_t ring = (size_t)q.stages * stage;
  const size_t scratch = tc_scratch_bytes(q.tn, q.splits, q.vec, split_rows_max(q.splits));
  q.smem = 1024 + tc_res_offset((uint32_t)ring, (uint32_t)scratch) + q.res_bytes + 256 + 16 + (size_t)q.tn * 4 * 10;
}

// Split-K policy for the HBM-bound regime: enough CTAs that every SM streams
// weights (>= one per SM), at most one resident wave, >= 2 k-blocks per CTA,
// cluster size <= 8 (portable).
static TcPlan plan(int M, int N, int K, int epi) {
  TcPlan q;
  q.tn = tn_for(M);
  q.n_tiles_n = (N + TC_BM - 1) / TC_BM;
  q.m_tiles = (M + q.tn - 1) / q.tn;
  const unsigned long long key = tune_key(q.tn, q.m_tiles, N, K);  // tuned entries are keyed by the default tile
  q.kb = (K + TC_BK - 1) / TC_BK;
  q.ctas_per_sm = g_tune_cps ? g_tune_cps : (q.tn >= 128 ? 1 : 2);
  // cps 3 (tuning only): size the grid for ONE CTA per SM but keep the smem of
  // two, leaving each SM a free slot for the next kernel's early weight prefetch (PDL)
  bool half_smem = (g_gemm_dbg & 32) != 0;  // experiment: every GEMM CTA fits beside another one (PDL prefetch)
  if (q.ctas_per_sm == 3) {
    q.ctas_per_sm = 1;
    half_smem = true;
  }
  int tuned_splits = 0, tuned_wt = 0, tuned_tn = 0;
  if (!g_tune_cps && !g_tune_splits) {
    std::lock_guard<std::mutex> lk(g_tuned_mu);
    auto it = g_tuned.find(key);
    if (it != g_tuned.end()) {
      q.ctas_per_sm = it->second.cps;
      tuned_splits = it->second.splits;
      tuned_wt = it->second.wt;
      tuned_tn = it->second.tn;
    }
  }
  // a narrower token tile (more, smaller CTAs: wave quantisation of the compute-bound regime)
  const int tn_over = g_tune_tn ? g_tune_tn : tuned_tn;
  if (tn_over >= 16 && tn_over < q.tn && tn_over % 16 == 0) {
    q.tn = tn_over;
    q.m_tiles = (M + q.tn - 1) / q.tn;
  }
  const int sms = num_sms();
  const int slots = sms * q.ctas_per_sm;
  const int tiles = q.n_tiles_n * q.m_tiles;
  // K splits (= cluster size; powers of two: measured, 3-CTA clusters and
  // multi-wave splits both lost 5-50% on B200): enough CTAs that every SM
  // streams, at most one resident wave, >= 2 k-blocks per CTA
  q.splits = 1;
  while (q.splits < 8 && tiles * q.splits < sms && tiles * q.splits * 2 <= slots && q.kb / (q.splits * 2) >= 2)
    q.splits *= 2;
  if (tuned_splits) q.splits = tuned_splits;
  if (g_tune_splits) q.splits = g_tune_splits;
  if (epi == EPI_ARGMAX) q.splits = 1;  // the fused argmax reads whole tiles straight from TMEM
  // large token tiles: two 128-row weight tiles per CTA share every X stage
  // (halves the L2->smem token traffic per FLOP; compute-bound regime)
  q.wt = 1;
  if (q.splits == 1 && q.ctas_per_sm == 1 && q.n_tiles_n >= 2 &&
      (tuned_wt ? tuned_wt == 2 : (q.tn >= 128 && (q.n_tiles_n + 1) / 2 * q.m_tiles >= sms)))
    q.wt = 2;  // (heuristic: only when the halved grid still covers every SM)
  if (g_tune_wt) q.wt = (q.splits == 1 && q.ctas_per_sm == 1 && q.n_tiles_n >= 2) ? g_tune_wt : 1;
  size_t budget = (q.ctas_per_sm == 2 || half_smem) ? 108 * 1024 : 200 * 1024;
  size_t stage = (size_t)(TC_BM * q.wt + q.tn) * TC_BK * 2;
  q.stages = (int)((budget - 1024 - 256) / stage);
  if (q.stages > (g_tune_stages ? g_tune_stages : 12)) q.stages = g_tune_stages ? g_tune_stages : 12;
  if (q.stages < 2) q.stages = 2;
  q.vec = 0;
  q.res_bytes = 0;
  tc_plan_smem(q);
  return q;
}

// Bulk-copy epilogue eligibility (16-byte rows, aligned outputs, power-of-two split ranks) and the
// residual prefetch of EPI_RESID_ADD (when this CTA's rows fit in 32 KB).
static void tc_plan_vec(TcPlan& q, const GemmArgs& a) {
  q.vec = !(g_gemm_dbg & 16) && a.N % 16 == 0 && !(q.splits & (q.splits - 1)) && !((uintptr_t)a.y & 15) &&
          !(a.out_xb && ((uintptr_t)a.out_xb & 15)) && !(a.bias && ((uintptr_t)a.bias & 7)) &&
          !(a.out_gain && ((uintptr_t)a.out_gain & 7));
  q.res_bytes = 0;
  if (q.vec && a.epi == EPI_RESID_ADD) {
    const int tok = q.splits > 1 ? (q.tn + q.splits - 1) / q.splits : q.tn;
    const int bytes = q.wt * tok * TC_BM * 4;
    if (bytes <= 32 * 1024) q.res_bytes = bytes;
  }
  tc_plan_smem(q);
  if (q.res_bytes && (q.smem > 220 * 1024 || (q.ctas_per_sm >= 2 && q.smem > 110 * 1024))) {
    // (within the kernel's smem limit, and two CTAs per SM stay resident)
    q.res_bytes = 0;
    tc_plan_smem(q);
  }
}

int gemm_tc_tune(int cps, int stages, int splits) {
  g_tune_cps = cps;
  g_tune_stages = stages;
  g_tune_splits = splits;
  return 0;
}

// Time the candidate (CTAs per SM, splits) configurations of one GEMM shape
// on real operands (EPI_STORE_F32 into y) and remember the fastest.
int gemm_tc_autotune(const void* x, const void* w, float* y, int M, int N, int K, cudaStream_t st, int* cps_out,
                     int* splits_out, float* us_out) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return SB_EINVAL;
  GemmArgs a{SB_BF16, x, w, y, M, N, K, K, EPI_STORE_F32, nullptr, 0};
  if (!gemm_tc_supported(a)) return SB_EUNSUPPORTED;
  const int save_cps = g_tune_cps, save_st = g_tune_stages, save_sp = g_tune_splits;
  const int kb = (K + TC_BK - 1) / TC_BK;
  const int tn = tn_for(M), m_tiles = (M + tn - 1) / tn;
  const int tiles = ((N + TC_BM - 1) / TC_BM) * m_tiles;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  int best_cps = 0, best_sp = 0, best_wt = 1, best_tn = 0, rc = 0;
  struct Cand {
    int cps, sp, wt, tn;
  };
  Cand cands[48];
  int nc = 0;
  // token tiles: the default, and for wide M the 128 / 192 tiles (more CTAs per wave)
  int tns[4] = {0, 0, 0, 0}, ntn = 1;
  if (M > 128 && tn > 128) tns[ntn++] = 128;
  if (M > 192 && tn > 192) tns[ntn++] = 192;
  {  // balanced tiles (e.g. 288 = 2 x 144, not 256 + 32): no mostly-empty remainder tile re-streaming weights
    const int nt = (M + TC_MAX_TN - 1) / TC_MAX_TN;
    const int tb = ((M + nt - 1) / nt + 15) / 16 * 16;
    if (nt == 2 && tb < tn && tb != 128 && tb != 192) tns[ntn++] = tb;  // (measured: T=288 7.8 -> 7.2 ms)
  }
  for (int ti = 0; ti < ntn; ++ti) {
    const int tn_c = tns[ti] ? tns[ti] : tn;
    const int tiles_c = ((N + TC_BM - 1) / TC_BM) * ((M + tn_c - 1) / tn_c);
    for (int cps = 1; cps <= 2; ++cps)
      for (int sp = 1; sp <= 8; sp *= 2) {
        if (sp > 1 && kb / sp < 2) break;
        if (tiles_c * sp > 2 * num_sms() * cps) break;  // more than two waves: never the winner
        cands[nc++] = {cps, sp, 1, tns[ti]};
      }
    if (tn_c >= 64 && (N + TC_BM - 1) / TC_BM >= 2) cands[nc++] = {1, 1, 2, tns[ti]};
  }
  for (int ci = 0; ci < nc && !rc; ++ci) {
    {
      const int cps = cands[ci].cps, sp = cands[ci].sp;
      g_tune_cps = cps;
      g_tune_splits = sp;
      g_tune_wt = cands[ci].wt;
      g_tune_tn = cands[ci].tn;
      g_tune_stages = 0;
      rc = gemm_tc(a, st);  // warm
      if (rc) break;
      const int reps = 5;
      cudaEventRecord(e0, st);
      for (int r = 0; r < reps && !rc; ++r) rc = gemm_tc(a, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const float us = ms * 1e3f / reps;
      if (!rc && us < best) {
        best = us;
        best_cps = cps;
        best_sp = sp;
        best_wt = cands[ci].wt;
        best_tn = cands[ci].tn;
      }
    }
  }
  g_tune_wt = 0;
  g_tune_tn = 0;
  g_tune_cps = save_cps;
  g_tune_stages = save_st;
  g_tune_splits = save_sp;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc) return rc;
  {
    std::lock_guard<std::mutex> lk(g_tuned_mu);
    g_tuned[tune_key(tn, m_tiles, N, K)] = {best_cps, best_sp, best_wt, best_tn};
  }
  if (cps_out) *cps_out = best_cps;
  if (splits_out) *splits_out = best_sp;
  if (us_out) *us_out = best;
  return 0;
}

int gemm_tc_tune_get(int M, int N, int K, int* cps, int* splits, int* wt, int* tn_out) {
  if (M <= 0 || N <= 0 || K <= 0) return SB_EINVAL;
  const int tn = tn_for(M), m_tiles = (M + tn - 1) / tn;
  std::lock_guard<std::mutex> lk(g_tuned_mu);
  auto it = g_tuned.find(tune_key(tn, m_tiles, N, K));
  if (it == g_tuned.end()) return SB_EINVAL;
  if (cps) *cps = it->second.cps;
  if (splits) *splits = it->second.splits;
  if (wt) *wt = it->second.wt;
  if (tn_out) *tn_out = it->second.tn;
  return 0;
}

int gemm_tc_tune_set(int M, int N, int K, int cps, int splits, int wt, int tn_set) {
  if (M <= 0 || N <= 0 || K <= 0 || cps < 1 || cps > 3 || splits < 1 || splits > 8 || wt < 1 || wt > 2 ||
      tn_set < 0 || tn_set > TC_MAX_TN || tn_set % 16)
    return SB_EINVAL;
  const int tn = tn_for(M), m_tiles = (M + tn - 1) / tn;
  std::lock_guard<std::mutex> lk(g_tuned_mu);
  g_tuned[tune_key(tn, m_tiles, N, K)] = {cps, splits, wt, tn_set};
  return 0;
}

int gemm_tc_autotune_clear() {
  std::lock_guard<std::mutex> lk(g_tuned_mu);
  g_tuned.clear();
  return 0;
}

// One instantiation per epilogue kind and style: each carries only its own epilogue code (the
// all-in-one kernel was 173 KB of SASS; its cold epilogue paths missed in the instruction cache
// under the saturated weight stream -- ncu: stall_no_inst / branch_resolving in the epilogue).
typedef void (*TcKernel)(CUtensorMap, CUtensorMap, TcParams);
static TcKernel tc_kernel_for(int epi, int vec) {
  static const TcKernel k[5][2] = {
      {gemm_tc_kernel<EPI_STORE, 0>, gemm_tc_kernel<EPI_STORE, 1>},
      {gemm_tc_kernel<EPI_STORE_F32, 0>, gemm_tc_kernel<EPI_STORE_F32, 1>},
      {gemm_tc_kernel<EPI_RESID_ADD, 0>, gemm_tc_kernel<EPI_RESID_ADD, 1>},
      {gemm_tc_kernel<EPI_SILU_MUL, 0>, gemm_tc_kernel<EPI_SILU_MUL, 1>},
      {gemm_tc_kernel<EPI_ARGMAX, 0>, gemm_tc_kernel<EPI_ARGMAX, 1>},
  };
  return k[epi < 0 || epi > 4 ? 1 : epi][vec ? 1 : 0];
}

int gemm_tc_init() {
  static int rc = -1;
  if (rc < 0) {
    cudaError_t e = cudaSuccess;
    for (int ep = 0; ep < 5 && e == cudaSuccess; ++ep)
      for (int v = 0; v < 2 && e == cudaSuccess; ++v)
        e = cudaFuncSetAttribute(tc_kernel_for(ep, v), cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    rc = (e == cudaSuccess) ? 0 : (int)e;
    if (!rc) rc = attention_tc_init();
    num_sms();
    get_encode();
  }
  return rc;
}

int gemm_tc_norm_partials(const GemmArgs& a) {
  TcPlan q = plan(a.M, a.N, a.K, a.epi);
  tc_plan_vec(q, a);
  return q.vec ? q.n_tiles_n : q.n_tiles_n * q.splits;  // row epilogue: one complete partial per tile
}

bool gemm_tc_supported(const GemmArgs& a) {
  if (a.dtype != SB_BF16) return false;
  if (a.K % 8 || a.ldx % 8) return false;  // 16-byte TMA strides
  if (((uintptr_t)a.x & 15) || ((uintptr_t)a.w & 15)) return false;
  if (a.epi == EPI_SILU_MUL && (a.N & 1)) return false;
  return get_encode() != nullptr;
}

size_t gemm_workspace_bytes(int, int, int) { return 0; }  // split-K reduces in DSMEM: no global scratch

int gemm_tc(const GemmArgs& a, cudaStream_t st) {
  if (!gemm_tc_supported(a)) return SB_EUNSUPPORTED;
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return SB_EINVAL;
  SB_TRY(gemm_tc_init());
  TcPlan q = plan(a.M, a.N, a.K, a.epi);
  tc_plan_vec(q, a);
  CUtensorMap mw, mx;
  SB_TRY(make_map(&mw, a.w, a.N, a.K, a.K, TC_BM * q.wt));
  SB_TRY(make_map(&mx, a.x, a.M, a.K, a.ldx, q.tn));
  TcParams p;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.tn = q.tn;
  p.n_tiles_n = q.n_tiles_n;
  p.kb = q.kb;
  p.splits = q.splits;
  p.wt = q.wt;
  p.stages = q.stages;
  p.epi = a.epi;
  p.y = a.y;
  p.aux_val = a.aux_val;
  p.aux_idx = a.aux_idx;
  p.ns_part = a.ns_part;
  p.ns_P = a.ns_P;
  p.ns_stride = a.ns_stride;
  p.ns_row_step = a.ns_row_step;
  p.ns_row_off = a.ns_row_off;
  p.ns_eps = a.ns_eps;
  p.ns_inv_h = a.ns_inv_h;
  p.out_part = a.out_part;
  p.out_xb = (__nv_bfloat16*)a.out_xb;
  p.out_gain = (const __nv_bfloat16*)a.out_gain;
  p.bias = (const __nv_bfloat16*)a.bias;
  p.relu = a.relu;
  p.pre_max = g_gemm_pre_max;
  p.launch_late = g_gemm_launch_late;
  p.dbg = g_gemm_dbg;
  p.ln_s1 = a.ln_s1;
  p.ln_c1 = a.ln_c1;
  p.ln_c2 = a.ln_c2;
  p.out_part1 = a.out_part1;
  if ((a.ln_s1 || a.ln_c1 || a.out_part1) && !q.vec) return SB_EUNSUPPORTED;  // row epilogue only
  if (a.ln_s1 && (!a.ln_c1 || !a.ln_c2 || !a.ns_part)) return SB_EINVAL;
  p.vec = q.vec;
  p.res_bytes = q.res_bytes;
  p.trace = g_cta_trace;
  p.trace_id = g_cta_trace ? g_cta_trace_seq++ : 0;
  if ((a.bias || a.relu) && (a.epi == EPI_SILU_MUL || a.epi == EPI_ARGMAX)) return SB_EINVAL;
  if (a.out_part && a.epi != EPI_RESID_ADD) return SB_EINVAL;
  if (a.epi == EPI_ARGMAX && (!a.aux_val || !a.aux_idx)) return SB_EINVAL;
  cudaLaunchConfig_t cfg = {};
  static int m_fast = -1;  // env SB_GEMM_MFAST
  if (m_fast < 0) {
    const char* e = getenv("SB_GEMM_MFAST");
    m_fast = e ? atoi(e) : 1;  // measured: prefill 21.9 -> 21.4 ms, T=288 verify 10.7 -> 10.4 ms
  }
  p.m_fast = m_fast && q.m_tiles > 1;
  static int k_rot = -1;  // env SB_GEMM_KROT
  if (k_rot < 0) {
    const char* e = getenv("SB_GEMM_KROT");
    k_rot = e ? atoi(e) : 1;  // measured: verify b=8,k=3 3.41 -> 3.35 ms, b=16,k=3 4.40 -> 4.30 ms
  }
  p.k_rot = k_rot;
  static int w_hint_env = -2;  // env SB_GEMM_W_L2HINT overrides the forward's choice (0/1/2)
  if (w_hint_env == -2) {
    const char* e = getenv("SB_GEMM_W_L2HINT");
    w_hint_env = e ? atoi(e) : -1;
  }
  p.w_hint = w_hint_env >= 0 ? w_hint_env : g_w_l2_hint;
  p.m_tiles = q.m_tiles;
  cfg.gridDim = p.m_fast ? dim3((q.n_tiles_n + q.wt - 1) / q.wt * q.splits * q.m_tiles, 1, 1)
                         : dim3((q.n_tiles_n + q.wt - 1) / q.wt * q.splits, q.m_tiles, 1);
  cfg.blockDim = dim3(TC_THREADS, 1, 1);
  cfg.dynamicSmemBytes = q.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = q.splits;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  if (g_pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_kernel_for(a.epi, q.vec), mw, mx, p);
  if (e != cudaSuccess) return (int)e;
  g_kernel_count++;
  return 0;
}

}  // namespace sb
