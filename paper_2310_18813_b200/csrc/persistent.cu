// Persistent decoder forward (bf16, T <= 256 query tokens): ONE kernel per
// forward of the draft step (K1) or the target verify (K2 + K3).
//
// Why: at decode sizes every GEMM of the layer stack is a weight stream
// (T = b(k+1) <= 72 tokens against 4096..22016-row weights) and the launch /
// pipeline-fill / tail of ~160 separate kernels per 7B forward costs ~35% of
// the HBM roofline.  Here one CTA per SM runs the whole forward:
//
//   phase 0            embedding gather (+ sum of squares for the fused norm)
//   per layer l        qkv GEMM (1/rms, RoPE, KV append in the epilogue)
//                      attention (flash decoding, causal inside the window)
//                      o GEMM (+residual, bf16 copy, norm partials)
//                      gate/up GEMM (silu(g)*u)
//                      down GEMM (+residual, bf16 copy, norm partials)
//   lm_head GEMM       fp32 logits and/or per-128-row argmax partials
//   finalize           greedy token per row -> token sink
//
// Phases are separated by a grid barrier (one counter in global memory), but
// the WEIGHT stream never waits for it: the weight producer warp runs ahead
// through all phases, bounded only by the shared-memory ring, so the next
// GEMM's weights are already in flight while the previous phase drains.  Only
// the activation (X) loads wait for the barrier.
//
// GEMMs are swap-AB tcgen05 (weight rows = UMMA_M 128, tokens = UMMA_N),
// accumulators double-buffered in TMEM, work split STREAM-K: the
// (tile, k-block) space of each GEMM is cut into equal contiguous ranges, one
// per CTA.  A tile cut between CTAs is finished by the CTA holding its first
// k-block (the "owner"; that segment is the LAST one it processes), which adds
// the other contributors' fp32 partials (published with release flags) in
// CTA order -- deterministic, no atomics on data.
//
// Warp roles (224 threads): w0 weight TMA producer, w1 TMEM allocator + MMA
// issuer, w2..w5 epilogue / attention / elementwise phases, w6 activation TMA
// producer (waits on the grid barrier).
#include <cuda.h>

#include <climits>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"
#include "mma_ptx.cuh"
#include "tc_ptx.cuh"

namespace sb {

constexpr int PK_THREADS = 224;
constexpr int PK_MAX_T = 256;
constexpr int PK_MAX_G = 1024;
constexpr int PK_ATT_KT = 64;
constexpr int PK_ATT_STAGES = 2;
constexpr int PK_STAGE_PAD = 17;  // RoPE staging row stride (floats)

enum : int { PG_QKV = 0, PG_O = 1, PG_GU = 2, PG_DOWN = 3, PG_LM = 4 };
enum : int { PH_EMBED = 0, PH_GEMM = 1, PH_ATTN = 2, PH_FINAL = 3 };

struct PkGemm {
  int N, K, kb, n_tiles, units, ctas;
};

struct PkParams {
  int T, n_seq, q_len, H, nq, nkv, hd, ffn, V, L;
  int tn, G, n_phases, stages;
  int lm_rows, lm_step, lm_off;
  int want_logits, want_argmax;
  float eps, inv_h, att_scale;
  int max_pos, ctx_max, kv_slots;
  PkGemm g[5];
  const int32_t* ids;
  const int32_t* slot;
  const int32_t* pos;
  const __nv_bfloat16* embed;
  const CUtensorMap* wmaps;  // [4L + 1] in global memory: per layer qkv, o, gu, down; then lm_head
  const float* cosT;
  const float* sinT;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  size_t layer_kv;  // elements per layer of the K (or V) cache
  float* resid;
  __nv_bfloat16* xb;
  __nv_bfloat16* qr;
  __nv_bfloat16* attn;
  __nv_bfloat16* act;
  float* npart;
  float* logits;
  float* amax_val;
  int* amax_idx;
  float* scratch;   // [G][tn][128] stream-K partial tiles
  unsigned* sync;   // [0] barrier counter, [1] exit counter, [2 .. 2+G) partial-ready flags
  int32_t* out_tok;
  int out_stride;
  int32_t* next_ids;
  int32_t* next_pos;
  const int32_t* base_pos;
  int pos_offset;
};

// ------------------------------------------------------------------ sync helpers
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
__device__ __noinline__ void wait_geq(const unsigned* p, unsigned target) {
  if (ld_acquire_u32(p) >= target) return;
  const uint64_t t0 = globaltimer();
  while (ld_acquire_u32(p) < target) {
    __nanosleep(32);
    if (globaltimer() - t0 > 20000000000ull) __trap();  // 20 s
  }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) { mbar_expect_tx(bar, bytes); }
__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float pk_silu(float g) { return g / (1.f + __expf(-g)); }

// ------------------------------------------------------------------ phase table
__device__ __forceinline__ int phase_kind(const PkParams& p, int ph, int& layer, int& gk) {
  layer = 0;
  gk = 0;
  if (ph == 0) return PH_EMBED;
  int q = ph - 1;
  if (q < 5 * p.L) {
    layer = q / 5;
    const int r = q % 5;
    if (r == 1) return PH_ATTN;
    gk = r == 0 ? PG_QKV : (r == 2 ? PG_O : (r == 3 ? PG_GU : PG_DOWN));
    return PH_GEMM;
  }
  if (q == 5 * p.L && p.lm_rows > 0) {
    layer = p.L;
    gk = PG_LM;
    return PH_GEMM;
  }
  return PH_FINAL;
}
__device__ __forceinline__ void unit_range(const PkGemm& g, int c, int& s, int& e) {
  if (c >= g.ctas) {
    s = e = 0;
    return;
  }
  s = (int)((long long)c * g.units / g.ctas);
  e = (int)((long long)(c + 1) * g.units / g.ctas);
}
__device__ __forceinline__ int unit_start(const PkGemm& g, int c) { return (int)((long long)c * g.units / g.ctas); }
__device__ __forceinline__ const CUtensorMap* wmap_of(const PkParams& p, int layer, int gk) {
  return gk == PG_LM ? p.wmaps + 4 * p.L : p.wmaps + 4 * layer + gk;
}

struct PkSmem {
  uint8_t* ring;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint32_t* tmem_slot;
  float* inv_s;   // [256]
  int* s_pos;     // [256]
  int* s_slot;    // [256]
  uint8_t* epi;   // aliased epilogue region (attention ring / RoPE staging / quadrant partials)
};

// ------------------------------------------------------------------ attention item
// One (sequence, kv head, 16-query chunk): S = Q K^T and O += P V with
// mma.sync m16n8k16 over 64-key tiles (warp w owns keys [16w, 16w+16) of each
// tile; warps combined in order).  Q is already rotated (qkv epilogue) and the
// window's K/V rows are already in the cache.
template <int HD>
__device__ void attn_item(const PkParams& p, uint8_t* epi, int seq, int kvh, int chunk, int* qpos, int* qtok,
                          int* qhead) {
  constexpr int RS = HD + 8, HALF = HD / 2, KSTEP = HD / 16, NT = HD / 8;
  constexpr size_t TILE = (size_t)PK_ATT_KT * RS * 2;
  constexpr size_t STAGE = 2 * TILE;
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(epi);
  uint8_t* ring = epi + (size_t)16 * RS * 2;
  const int tid = threadIdx.x - 64, warp = tid >> 5, lane = tid & 31;
  const int group = p.nq / p.nkv;
  const int nQ = group * p.q_len;
  const int slot = p.slot[seq];
  const __nv_bfloat16* kslab = p.kc + ((size_t)slot * p.nkv + kvh) * p.ctx_max * HD;
  const __nv_bfloat16* vslab = p.vc + ((size_t)slot * p.nkv + kvh) * p.ctx_max * HD;
  (void)HALF;
  if (tid < 16) {
    const int jj = chunk * 16 + tid;
    const int t = jj / group;
    const bool ok = jj < nQ;
    qtok[tid] = ok ? t : 0;
    qhead[tid] = kvh * group + (ok ? jj % group : 0);
    qpos[tid] = ok ? p.pos[seq * p.q_len + t] : -1;
  }
  epi_sync();
  const int qd = p.nq * HD;
  for (int e = tid; e < 16 * (HD / 8); e += 128) {
    const int j = e / (HD / 8), c = (e % (HD / 8)) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (qpos[j] >= 0)
      v = __ldcg(reinterpret_cast<const uint4*>(p.qr + (size_t)(seq * p.q_len + qtok[j]) * qd + qhead[j] * HD + c));
    *reinterpret_cast<uint4*>(Qs + j * RS + c) = v;
  }
  epi_sync();
  int maxp = -1;
#pragma unroll
  for (int j = 0; j < 16; ++j) maxp = max(maxp, qpos[j]);
  const int n_keys = maxp + 1;
  const int n_tiles = (n_keys + PK_ATT_KT - 1) / PK_ATT_KT;

  auto issue = [&](int tile) {
    if (tile < n_tiles) {
      uint8_t* st = ring + (tile % PK_ATT_STAGES) * STAGE;
      __nv_bfloat16* Kd = reinterpret_cast<__nv_bfloat16*>(st);
      __nv_bfloat16* Vd = reinterpret_cast<__nv_bfloat16*>(st + TILE);
      const int k0 = tile * PK_ATT_KT;
      constexpr int CPR = HD / 8;
      for (int e = tid; e < PK_ATT_KT * CPR; e += 128) {
        const int r = e / CPR, c = (e % CPR) * 8;
        const int key = k0 + r;
        if (key < n_keys) {
          cp_async16(Kd + r * RS + c, kslab + (size_t)key * HD + c);
          cp_async16(Vd + r * RS + c, vslab + (size_t)key * HD + c);
        } else {
          *reinterpret_cast<uint4*>(Kd + r * RS + c) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(Vd + r * RS + c) = make_uint4(0, 0, 0, 0);
        }
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int i = 0; i < PK_ATT_STAGES - 1; ++i) issue(i);

  const uint32_t qs_base = (uint32_t)__cvta_generic_to_shared(Qs);
  uint32_t qa[KSTEP][4];
  {
    const int mi = lane >> 3, ri = lane & 7;
    const int row = ri + (mi & 1) * 8;
#pragma unroll
    for (int ks = 0; ks < KSTEP; ++ks) {
      const int col = ks * 16 + (mi >> 1) * 8;
      ldsm_x4(qs_base + (uint32_t)(row * RS + col) * 2, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
  }
  const int g = lane >> 2, t4 = lane & 3;
  const int pos_lo = qpos[g], pos_hi = qpos[g + 8];
  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
  const float scale = p.att_scale;

  for (int tile = 0; tile < n_tiles; ++tile) {
    issue(tile + PK_ATT_STAGES - 1);
    cp_async_wait<PK_ATT_STAGES - 1>();
    epi_sync();
    const uint8_t* st = ring + (tile % PK_ATT_STAGES) * STAGE;
    const uint32_t kb = (uint32_t)__cvta_generic_to_shared(st);
    const uint32_t vb = kb + (uint32_t)TILE;
    const int kw = warp * 16;
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const int mi = lane >> 3, ri = lane & 7;
      const int key = kw + ri + (mi >> 1) * 8;
#pragma unroll
      for (int ks = 0; ks < KSTEP; ++ks) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kb + (uint32_t)(key * RS + ks * 16 + (mi & 1) * 8) * 2, b0, b1, b2, b3);
        mma_bf16(s0, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
        mma_bf16(s1, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
      }
    }
    const int kbase = tile * PK_ATT_KT + kw + 2 * t4;
    float v[8] = {s0[0], s0[1], s1[0], s1[1], s0[2], s0[3], s1[2], s1[3]};
    const int kidx[4] = {kbase, kbase + 1, kbase + 8, kbase + 9};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = (kidx[i] <= pos_lo) ? v[i] * scale : -INFINITY;
      v[4 + i] = (kidx[i] <= pos_hi) ? v[4 + i] * scale : -INFINITY;
    }
    float mx_lo = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
    float mx_hi = fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7]));
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
    const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
    const float c_lo = (m_lo == -INFINITY) ? 0.f : __expf(m_lo - mn_lo);
    const float c_hi = (m_hi == -INFINITY) ? 0.f : __expf(m_hi - mn_hi);
    float pr[8], sum_lo = 0.f, sum_hi = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      pr[i] = (mn_lo == -INFINITY) ? 0.f : __expf(v[i] - mn_lo);
      pr[4 + i] = (mn_hi == -INFINITY) ? 0.f : __expf(v[4 + i] - mn_hi);
      sum_lo += pr[i];
      sum_hi += pr[4 + i];
    }
    sum_lo += __shfl_xor_sync(0xffffffffu, sum_lo, 1);
    sum_lo += __shfl_xor_sync(0xffffffffu, sum_lo, 2);
    sum_hi += __shfl_xor_sync(0xffffffffu, sum_hi, 1);
    sum_hi += __shfl_xor_sync(0xffffffffu, sum_hi, 2);
    l_lo = l_lo * c_lo + sum_lo;
    l_hi = l_hi * c_hi + sum_hi;
    m_lo = mn_lo;
    m_hi = mn_hi;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      o[n][0] *= c_lo;
      o[n][1] *= c_lo;
      o[n][2] *= c_hi;
      o[n][3] *= c_hi;
    }
    const uint32_t pa0 = pack_bf16(pr[0], pr[1]), pa1 = pack_bf16(pr[4], pr[5]);
    const uint32_t pa2 = pack_bf16(pr[2], pr[3]), pa3 = pack_bf16(pr[6], pr[7]);
    {
      const int mi = lane >> 3, ri = lane & 7;
      const int key = kw + ri + (mi & 1) * 8;
#pragma unroll
      for (int n = 0; n < NT; n += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vb + (uint32_t)(key * RS + n * 8 + (mi >> 1) * 8) * 2, b0, b1, b2, b3);
        mma_bf16(o[n], pa0, pa1, pa2, pa3, b0, b1);
        mma_bf16(o[n + 1], pa0, pa1, pa2, pa3, b2, b3);
      }
    }
    epi_sync();
  }
  cp_async_wait<0>();
  epi_sync();
  float* comb = reinterpret_cast<float*>(ring);
  float* cm = comb + 4 * 16 * HD;
  float* cl = cm + 4 * 16;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int d = n * 8 + 2 * t4;
    comb[(warp * 16 + g) * HD + d] = o[n][0];
    comb[(warp * 16 + g) * HD + d + 1] = o[n][1];
    comb[(warp * 16 + g + 8) * HD + d] = o[n][2];
    comb[(warp * 16 + g + 8) * HD + d + 1] = o[n][3];
  }
  if (t4 == 0) {
    cm[warp * 16 + g] = m_lo;
    cm[warp * 16 + g + 8] = m_hi;
    cl[warp * 16 + g] = l_lo;
    cl[warp * 16 + g + 8] = l_hi;
  }
  epi_sync();
  for (int e = tid; e < 16 * HD; e += 128) {
    const int j = e / HD, d = e % HD;
    if (qpos[j] < 0) continue;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, cm[w * 16 + j]);
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = cm[w * 16 + j];
      const float f = (mw == -INFINITY) ? 0.f : __expf(mw - M);
      L += cl[w * 16 + j] * f;
      acc += comb[(w * 16 + j) * HD + d] * f;
    }
    p.attn[((size_t)(seq * p.q_len + qtok[j]) * p.nq + qhead[j]) * HD + d] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
  }
  epi_sync();  // the ring / comb region is reused by the next item
}

// ------------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(PK_THREADS, 1)
    persistent_forward_kernel(const __grid_constant__ CUtensorMap map_xb, const __grid_constant__ CUtensorMap map_attn,
                              const __grid_constant__ CUtensorMap map_act, const __grid_constant__ CUtensorMap map_lm,
                              const __grid_constant__ PkParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int tn = p.tn, S = p.stages, G = p.G, c = blockIdx.x;
  const uint32_t a_bytes = TC_BM * TC_BK * 2;
  const uint32_t b_bytes = (uint32_t)tn * TC_BK * 2;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  PkSmem sm;
  sm.ring = base;
  size_t off = (size_t)S * stage_bytes;
  sm.epi = base + off;
  const size_t att_bytes = p.hd == 128 ? (size_t)16 * 136 * 2 + (size_t)PK_ATT_STAGES * 2 * PK_ATT_KT * 136 * 2
                                       : (size_t)16 * 72 * 2 + (size_t)PK_ATT_STAGES * 2 * PK_ATT_KT * 72 * 2;
  size_t epi_bytes = att_bytes;
  if ((size_t)128 * PK_STAGE_PAD * 4 > epi_bytes) epi_bytes = (size_t)128 * PK_STAGE_PAD * 4;
  if ((size_t)8 * tn * 4 > epi_bytes) epi_bytes = (size_t)8 * tn * 4;
  off += (epi_bytes + 127) & ~(size_t)127;
  sm.inv_s = (float*)(base + off);
  off += PK_MAX_T * 4;
  sm.s_pos = (int*)(base + off);
  off += PK_MAX_T * 4;
  sm.s_slot = (int*)(base + off);
  off += PK_MAX_T * 4;
  sm.full = (uint64_t*)(base + off);
  sm.empty = sm.full + S;
  sm.tfull = sm.empty + S;
  sm.tempty = sm.tfull + 2;
  sm.tmem_slot = (uint32_t*)(sm.tempty + 2);
  __shared__ int a_qpos[16], a_qtok[16], a_qhead[16];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < 2 * tn) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 2);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.tfull[b], 1);
      mbar_init(&sm.tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sm.tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sm.tmem_slot;
  unsigned* bar = p.sync;
  unsigned* done = p.sync + 1;
  unsigned* flags = p.sync + 2;

  if (warp == 0) {
    // ================= weight producer: runs ahead through every GEMM phase
    // (weights never depend on earlier phases, nor on the previous kernel)
    if (lane == 0) {
      uint32_t it = 0;
      for (int ph = 1; ph < p.n_phases; ++ph) {
        int layer, gk;
        if (phase_kind(p, ph, layer, gk) != PH_GEMM) continue;
        const PkGemm& g = p.g[gk];
        const CUtensorMap* wm = wmap_of(p, layer, gk);
        int s, e;
        unit_range(g, c, s, e);
        for (int u = s; u < e; ++u, ++it) {
          const int stg = (int)(it % S);
          if (it >= (uint32_t)S) mbar_wait(&sm.empty[stg], ((it / S) + 1) & 1);
          mbar_arrive_expect(&sm.full[stg], a_bytes);
          const int tile = u / g.kb, kbi = u - tile * g.kb;
          tma_load_2d(sm.ring + (size_t)stg * stage_bytes, wm, &sm.full[stg], kbi * TC_BK, tile * TC_BM);
        }
      }
    }
  } else if (warp == 6) {
    // ================= activation producer: X tiles of phase ph only after the
    // grid barrier says every CTA finished phases < ph
    if (lane == 0) {
      griddep_wait();
      uint32_t it = 0;
      for (int ph = 1; ph < p.n_phases; ++ph) {
        int layer, gk;
        if (phase_kind(p, ph, layer, gk) != PH_GEMM) continue;
        const PkGemm& g = p.g[gk];
        const CUtensorMap* xm = gk == PG_O ? &map_attn : (gk == PG_DOWN ? &map_act : (gk == PG_LM ? &map_lm : &map_xb));
        int s, e;
        unit_range(g, c, s, e);
        if (s < e) {
          wait_geq(bar, (unsigned)(ph * G));
          fence_proxy_async();
        }
        for (int u = s; u < e; ++u, ++it) {
          const int stg = (int)(it % S);
          if (it >= (uint32_t)S) mbar_wait(&sm.empty[stg], ((it / S) + 1) & 1);
          mbar_arrive_expect(&sm.full[stg], b_bytes);
          const int kbi = u % g.kb;
          tma_load_2d(sm.ring + (size_t)stg * stage_bytes + a_bytes, xm, &sm.full[stg], kbi * TC_BK, 0);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc(tn);
      uint32_t it = 0, seg = 0;
      for (int ph = 1; ph < p.n_phases; ++ph) {
        int layer, gk;
        if (phase_kind(p, ph, layer, gk) != PH_GEMM) continue;
        const PkGemm& g = p.g[gk];
        int s, e;
        unit_range(g, c, s, e);
        int u = s;
        while (u < e) {
          const int tile = u / g.kb;
          const int seg_end = min(e, (tile + 1) * g.kb);
          const int buf = seg & 1;
          const uint32_t use = seg >> 1;
          if (seg >= 2) mbar_wait(&sm.tempty[buf], (use + 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(buf * tn);
          const int first = u;
          for (; u < seg_end; ++u, ++it) {
            const int stg = (int)(it % S);
            mbar_wait(&sm.full[stg], (it / S) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(sm.ring + (size_t)stg * stage_bytes);
            const uint32_t sb = sa + a_bytes;
#pragma unroll
            for (int kk = 0; kk < TC_BK / TC_UK; ++kk)
              tc_mma(d, sw128_desc(sa + kk * TC_UK * 2), sw128_desc(sb + kk * TC_UK * 2), idesc,
                     (u > first || kk > 0) ? 1u : 0u);
            tc_commit(&sm.empty[stg]);
          }
          tc_commit(&sm.tfull[buf]);
          ++seg;
        }
      }
    }
  } else {
    // ================= epilogue / attention / elementwise warps (128 threads)
    griddep_wait();
    const int et = threadIdx.x - 64;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    const int T = p.T, H = p.H;
    const int nTH = (H + TC_BM - 1) / TC_BM;  // norm partials written by o / down
    uint32_t seg = 0;
    for (int ph = 0; ph < p.n_phases; ++ph) {
      int layer, gk;
      const int kind = phase_kind(p, ph, layer, gk);
      if (et == 0) wait_geq(bar, (unsigned)(ph * G));
      epi_sync();
      if (kind == PH_EMBED) {
        float* red = reinterpret_cast<float*>(sm.epi);
        for (int m = c; m < T; m += G) {
          const int id = p.ids[m];
          const bool pad = p.pos[m] < 0 || id < 0 || id >= p.V;
          const __nv_bfloat16* er = p.embed + (size_t)(pad ? 0 : id) * H;
          float ss = 0.f;
          for (int i = et; i < H; i += 128) {
            const float v = pad ? 0.f : __bfloat162float(er[i]);
            p.resid[(size_t)m * H + i] = v;
            p.xb[(size_t)m * H + i] = __float2bfloat16_rn(v);
            ss += v * v;
          }
          ss = warp_sum(ss);
          if (lane == 0) red[warp - 2] = ss;
          epi_sync();
          if (et == 0) p.npart[m] = ((red[0] + red[1]) + red[2]) + red[3];
          epi_sync();
        }
      } else if (kind == PH_ATTN) {
        const int group = p.nq / p.nkv;
        const int n_chunks = (group * p.q_len + 15) / 16;
        const int items = p.n_seq * p.nkv * n_chunks;
        for (int i = c; i < items; i += G) {
          const int chunk = i % n_chunks;
          const int kvh = (i / n_chunks) % p.nkv;
          const int seq = i / (n_chunks * p.nkv);
          if (p.hd == 128)
            attn_item<128>(p, sm.epi, seq, kvh, chunk, a_qpos, a_qtok, a_qhead);
          else
            attn_item<64>(p, sm.epi, seq, kvh, chunk, a_qpos, a_qtok, a_qhead);
        }
      } else if (kind == PH_FINAL) {
        const int nt = p.g[PG_LM].n_tiles;
        const int rows = p.lm_rows;
        const int wq = warp - 2;
        for (int r = c * 4 + wq; r < rows; r += G * 4) {
          ArgMax a{-INFINITY, INT_MAX};
          for (int t = lane; t < nt; t += 32)
            a = argmax_merge(a, ArgMax{__ldcg(&p.amax_val[(size_t)t * rows + r]), __ldcg(&p.amax_idx[(size_t)t * rows + r])});
          a = warp_argmax(a);
          if (lane == 0) {
            if (p.out_tok) p.out_tok[(size_t)r * p.out_stride] = a.i;
            if (p.next_ids) p.next_ids[r] = a.i;
            if (p.next_pos) p.next_pos[r] = p.base_pos[r] + p.pos_offset;
          }
        }
      } else {
        // ---------------- GEMM epilogue
        const PkGemm& g = p.g[gk];
        const int N = g.N;
        const bool norm_in = gk == PG_QKV || gk == PG_GU || gk == PG_LM;
        const int rows = gk == PG_LM ? p.lm_rows : T;
        int s, e;
        unit_range(g, c, s, e);
        if (s < e) {
          if (norm_in) {
            int P_in = nTH;
            int step = 1, roff = 0;
            if (gk == PG_QKV && layer == 0) P_in = 1;
            if (gk == PG_LM) {
              step = p.lm_step;
              roff = p.lm_off;
              if (p.L == 0) P_in = 1;
            }
            for (int j = et; j < tn; j += 128) {
              float sacc = 0.f;
              if (j < rows) {
                const float* src = p.npart + (size_t)j * step + roff;
                for (int q = 0; q < P_in; ++q) sacc += __ldcg(src + (size_t)q * T);
              }
              sm.inv_s[j] = rsqrtf(sacc * p.inv_h + p.eps);
            }
          }
          if (gk == PG_QKV) {
            for (int j = et; j < T; j += 128) {
              sm.s_pos[j] = p.pos[j];
              sm.s_slot[j] = p.slot[j / p.q_len];
            }
          }
          epi_sync();
        }
        int u = s;
        while (u < e) {
          const int tile = u / g.kb;
          const int a0 = u - tile * g.kb;
          const int seg_end = min(e, (tile + 1) * g.kb);
          const int b1 = seg_end - tile * g.kb;
          const bool contrib = a0 > 0;
          const bool owner = a0 == 0 && b1 < g.kb;
          const int buf = seg & 1;
          const uint32_t use = seg >> 1;
          const int n0 = tile * TC_BM;
          const int n = n0 + row;
          int c_last = c;
          if (owner) {
            while (c_last + 1 < g.ctas && unit_start(g, c_last + 1) < (tile + 1) * g.kb) ++c_last;
            if (et == 0)
              for (int c2 = c + 1; c2 <= c_last; ++c2) wait_geq(&flags[c2], (unsigned)(ph + 1));
          }
          mbar_wait(&sm.tfull[buf], use & 1);
          tc_fence_after();
          if (owner) epi_sync();
          // QKV tile region: 0 = Q, 1 = K, 2 = V (tiles never straddle: checked on the host)
          const int qd = p.nq * p.hd, kd = p.nkv * p.hd;
          const int region = n0 < qd ? 0 : (n0 < qd + kd ? 1 : 2);
          float* stage_f = reinterpret_cast<float*>(sm.epi);
          float* qv = reinterpret_cast<float*>(sm.epi);
          int* qi = reinterpret_cast<int*>(sm.epi) + 4 * tn;
          for (int j0 = 0; j0 < tn; j0 += 16) {
            float v[16];
            tmem_ld16(lane_addr + (uint32_t)(buf * tn + j0), v);
            if (contrib) {
              float* dst = p.scratch + ((size_t)c * tn + j0) * TC_BM + row;
#pragma unroll
              for (int j = 0; j < 16; ++j) dst[(size_t)j * TC_BM] = v[j];
              continue;
            }
            if (owner) {
              for (int c2 = c + 1; c2 <= c_last; ++c2) {
                const float* src = p.scratch + ((size_t)c2 * tn + j0) * TC_BM + row;
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] += __ldcg(src + (size_t)j * TC_BM);
              }
            }
            if (gk == PG_QKV) {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = bf16r(v[j] * sm.inv_s[j0 + j]);
              const int d = (n - (region == 0 ? 0 : (region == 1 ? qd : qd + kd))) % p.hd;
              const int head = (n - (region == 0 ? 0 : (region == 1 ? qd : qd + kd))) / p.hd;
              __nv_bfloat16* kv_base = (region == 1 ? p.kc : p.vc) + (size_t)layer * p.layer_kv;
              if (region < 2) {
                const int half = p.hd >> 1;
#pragma unroll
                for (int j = 0; j < 16; ++j) stage_f[row * PK_STAGE_PAD + j] = v[j];
                epi_sync();
                const bool lo = d < half;
                const int prow = lo ? row + half : row - half;
                const int di = lo ? d : d - half;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                  const int m = j0 + j;
                  if (m >= T || n >= N) continue;
                  const float xp = stage_f[prow * PK_STAGE_PAD + j];
                  const int ps = sm.s_pos[m];
                  const int pc = ps < 0 ? 0 : (ps >= p.max_pos ? p.max_pos - 1 : ps);
                  const float cs = p.cosT[(size_t)pc * half + di], sn = p.sinT[(size_t)pc * half + di];
                  const float r = lo ? v[j] * cs - xp * sn : v[j] * cs + xp * sn;
                  const __nv_bfloat16 ob = __float2bfloat16_rn(r);
                  if (region == 0) {
                    p.qr[(size_t)m * qd + n] = ob;
                  } else if (ps >= 0) {
                    kv_base[(((size_t)sm.s_slot[m] * p.nkv + head) * p.ctx_max + ps) * p.hd + d] = ob;
                  }
                }
                epi_sync();
              } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                  const int m = j0 + j;
                  if (m >= T || n >= N) continue;
                  const int ps = sm.s_pos[m];
                  if (ps >= 0)
                    kv_base[(((size_t)sm.s_slot[m] * p.nkv + head) * p.ctx_max + ps) * p.hd + d] =
                        __float2bfloat16_rn(v[j]);
                }
              }
            } else if (gk == PG_GU) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float x = v[j] * sm.inv_s[j0 + j];
                const float other = __shfl_xor_sync(0xffffffffu, x, 1);
                const int m = j0 + j;
                if (!(lane & 1) && m < T && n < N)
                  p.act[(size_t)m * (N / 2) + n / 2] = __float2bfloat16_rn(pk_silu(x) * other);
              }
            } else if (gk == PG_O || gk == PG_DOWN) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int m = j0 + j;
                float sq = 0.f;
                if (m < T && n < N) {
                  const size_t o = (size_t)m * H + n;
                  const float nv = __ldcg(&p.resid[o]) + v[j];
                  p.resid[o] = nv;
                  p.xb[o] = __float2bfloat16_rn(nv);
                  sq = nv * nv;
                }
                sq = warp_sum(sq);
                if (lane == 0) qv[quad * tn + j0 + j] = sq;
              }
            } else {  // PG_LM
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int m = j0 + j;
                const float x = v[j] * sm.inv_s[m];
                if (p.want_logits && m < rows && n < N) p.logits[(size_t)m * N + n] = x;
                if (p.want_argmax) {
                  ArgMax a = warp_argmax(ArgMax{n < N ? x : -INFINITY, n < N ? n : INT_MAX});
                  if (lane == 0) {
                    qv[quad * tn + m] = a.v;
                    qi[quad * tn + m] = a.i;
                  }
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.tempty[buf]);
          if (contrib) {
            epi_sync();
            if (et == 0) {
              __threadfence();
              st_release_u32(&flags[c], (unsigned)(ph + 1));
            }
          } else if (gk == PG_O || gk == PG_DOWN || (gk == PG_LM && p.want_argmax)) {
            epi_sync();
            for (int j = et; j < rows; j += 128) {
              if (gk == PG_LM) {
                ArgMax a{qv[j], qi[j]};
#pragma unroll
                for (int q = 1; q < 4; ++q) a = argmax_merge(a, ArgMax{qv[q * tn + j], qi[q * tn + j]});
                p.amax_val[(size_t)tile * rows + j] = a.v;
                p.amax_idx[(size_t)tile * rows + j] = a.i;
              } else {
                p.npart[(size_t)tile * T + j] = ((qv[j] + qv[tn + j]) + qv[2 * tn + j]) + qv[3 * tn + j];
              }
            }
            epi_sync();
          }
          u = seg_end;
          ++seg;
        }
      }
      // ---- phase done: publish (fence orders generic writes for other SMs' TMA reads)
      epi_sync();
      if (et == 0) {
        __threadfence();
        fence_proxy_async();
        atomicAdd(bar, 1u);
        if (ph == p.n_phases - 2) griddep_launch();
      }
    }
    // ---- exit protocol: the last CTA out resets the sync words for the next launch
    if (et == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(done, 1u);
      if (prev == (unsigned)G - 1) {
        for (int i = 0; i < G; ++i) flags[i] = 0;
        *bar = 0;
        __threadfence();
        *done = 0;
        __threadfence();
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
  }
}

// ------------------------------------------------------------------ host side
static int g_persistent = 1;  // sb_set_persistent

static size_t pk_epi_bytes(int hd, int tn) {
  const int RS = hd + 8;
  size_t att = (size_t)16 * RS * 2 + (size_t)PK_ATT_STAGES * 2 * PK_ATT_KT * RS * 2;
  size_t e = att;
  if ((size_t)128 * PK_STAGE_PAD * 4 > e) e = (size_t)128 * PK_STAGE_PAD * 4;
  if ((size_t)8 * tn * 4 > e) e = (size_t)8 * tn * 4;
  return (e + 127) & ~(size_t)127;
}

static int pk_grid() {
  static int g = 0;
  if (!g) {
    g = num_sms();
    if (g > PK_MAX_G) g = PK_MAX_G;
  }
  return g;
}

size_t persistent_sync_bytes() { return (size_t)(2 + PK_MAX_G) * 4; }
size_t persistent_scratch_bytes(int T) {
  const int tn = T <= 16 ? 16 : (T + 15) / 16 * 16;
  return (size_t)pk_grid() * (tn > 256 ? 256 : tn) * TC_BM * 4;
}

bool persistent_eligible(const sb_decoder_t* m, int T) {
  if (!g_persistent || m->dtype != SB_BF16 || !m->tmaps || T > PK_MAX_T) return false;
  if (m->head_dim != 64 && m->head_dim != 128) return false;
  const int qd = m->n_heads * m->head_dim, kd = m->n_kv_heads * m->head_dim;
  if (qd % TC_BM || kd % TC_BM) return false;
  if (m->hidden % 64 || m->ffn % 64 || qd % 64) return false;
  if (m->n_heads % m->n_kv_heads) return false;
  return true;
}

int persistent_forward(const sb_decoder_t* m, const sb_kvcache_t* kv, const int32_t* ids, const int32_t* slot,
                       const int32_t* pos, int n_seq, int q_len, float* logits, int logits_mode,
                       const sb_token_sink_t* sink, const PkBuffers& b, cudaStream_t st) {
  const int T = n_seq * q_len;
  PkParams p;
  memset(&p, 0, sizeof(p));
  p.T = T;
  p.n_seq = n_seq;
  p.q_len = q_len;
  p.H = m->hidden;
  p.nq = m->n_heads;
  p.nkv = m->n_kv_heads;
  p.hd = m->head_dim;
  p.ffn = m->ffn;
  p.V = m->vocab;
  p.L = m->n_layers;
  p.tn = T <= 16 ? 16 : (T + 15) / 16 * 16;
  p.G = pk_grid();
  const int qkv_n = (p.nq + 2 * p.nkv) * p.hd;
  const int qd = p.nq * p.hd;
  const bool want_lm = logits_mode != SB_LOGITS_NONE;
  const bool last = logits_mode == SB_LOGITS_LAST;
  p.lm_rows = want_lm ? (last ? n_seq : T) : 0;
  p.lm_step = last ? q_len : 1;
  p.lm_off = last ? q_len - 1 : 0;
  p.want_argmax = want_lm && sink != nullptr;
  p.want_logits = want_lm && logits != nullptr;
  if (want_lm && !p.want_argmax && !p.want_logits) return SB_EINVAL;
  p.n_phases = 1 + 5 * p.L + (want_lm ? 1 : 0) + (p.want_argmax ? 1 : 0);
  p.eps = m->rms_eps;
  p.inv_h = 1.0f / (float)p.H;
  p.att_scale = 1.0f / sqrtf((float)p.hd);
  p.max_pos = m->max_pos;
  p.ctx_max = kv->ctx_max;
  p.kv_slots = kv->slots;
  const int dims[5][2] = {{qkv_n, p.H}, {p.H, qd}, {2 * p.ffn, p.H}, {p.H, p.ffn}, {p.V, p.H}};
  for (int i = 0; i < 5; ++i) {
    PkGemm& g = p.g[i];
    g.N = dims[i][0];
    g.K = dims[i][1];
    g.kb = (g.K + TC_BK - 1) / TC_BK;
    g.n_tiles = (g.N + TC_BM - 1) / TC_BM;
    g.units = g.n_tiles * g.kb;
    // >= 4 k-blocks per CTA (fewer only spreads the fixed per-segment cost)
    int ctas = (g.units + 3) / 4;
    g.ctas = ctas < p.G ? ctas : p.G;
  }
  p.ids = ids;
  p.slot = slot;
  p.pos = pos;
  p.embed = (const __nv_bfloat16*)m->embed;
  p.wmaps = (const CUtensorMap*)m->tmaps;
  p.cosT = m->rope_cos;
  p.sinT = m->rope_sin;
  p.kc = (__nv_bfloat16*)kv->k;
  p.vc = (__nv_bfloat16*)kv->v;
  p.layer_kv = (size_t)kv->slots * p.nkv * kv->ctx_max * p.hd;
  p.resid = b.resid;
  p.xb = (__nv_bfloat16*)b.xb;
  p.qr = (__nv_bfloat16*)b.qr;
  p.attn = (__nv_bfloat16*)b.attn;
  p.act = (__nv_bfloat16*)b.act;
  p.npart = b.npart;
  p.logits = logits;
  p.amax_val = b.amax_val;
  p.amax_idx = b.amax_idx;
  p.scratch = b.scratch;
  p.sync = b.sync;
  if (sink) {
    p.out_tok = sink->out_tok;
    p.out_stride = sink->out_stride;
    p.next_ids = sink->next_ids;
    p.next_pos = sink->next_pos;
    p.base_pos = sink->base_pos;
    p.pos_offset = sink->pos_offset;
    if (p.next_pos && !p.base_pos) return SB_EINVAL;
  }
  // shared memory: ring gets what the epilogue region leaves
  const size_t epi = pk_epi_bytes(p.hd, p.tn);
  const size_t fixed = 1024 + epi + 3 * PK_MAX_T * 4 + 64 * 8 + 16;
  const size_t budget = 226 * 1024;
  const size_t stage = (size_t)(TC_BM + p.tn) * TC_BK * 2;
  int S = (int)((budget - fixed) / stage);
  if (S > 16) S = 16;
  if (S < 2) return SB_EUNSUPPORTED;
  p.stages = S;
  const size_t smem = 1024 + (size_t)S * stage + epi + 3 * PK_MAX_T * 4 + (2 * S + 4) * 8 + 16;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(persistent_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  CUtensorMap mx, ma, mc, ml;
  SB_TRY(make_map(&mx, b.xb, T, p.H, p.H, p.tn));
  SB_TRY(make_map(&ma, b.attn, T, qd, qd, p.tn));
  SB_TRY(make_map(&mc, b.act, T, p.ffn, p.ffn, p.tn));
  if (want_lm) {
    SB_TRY(make_map(&ml, (const char*)b.xb + (size_t)p.lm_off * p.H * 2, p.lm_rows, p.H, p.lm_step * p.H, p.tn));
  } else {
    ml = mx;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.G, 1, 1);
  cfg.blockDim = dim3(PK_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, persistent_forward_kernel, mx, ma, mc, ml, p);
  if (e != cudaSuccess) return (int)e;
  ++g_kernel_count;
  return 0;
}

int set_persistent(int enabled) {
  g_persistent = enabled ? 1 : 0;
  return 0;
}

// Weight tensor maps (global memory, encoded once per decoder): per layer
// qkv, o, gu, down, then lm_head.  Box 64 x 128 rows, 128B swizzle.
size_t decoder_tmaps_bytes(const sb_decoder_t* m) { return (size_t)(4 * m->n_layers + 1) * sizeof(CUtensorMap); }

int decoder_encode_tmaps(const sb_decoder_t* m, void* host_out) {
  if (m->dtype != SB_BF16) return SB_EUNSUPPORTED;
  CUtensorMap* o = (CUtensorMap*)host_out;
  const int H = m->hidden, qd = m->n_heads * m->head_dim;
  const int qkv_n = (m->n_heads + 2 * m->n_kv_heads) * m->head_dim;
  for (int l = 0; l < m->n_layers; ++l) {
    SB_TRY(make_map(&o[4 * l + 0], m->w_qkv[l], qkv_n, H, H, TC_BM));
    SB_TRY(make_map(&o[4 * l + 1], m->w_o[l], H, qd, qd, TC_BM));
    SB_TRY(make_map(&o[4 * l + 2], m->w_gu[l], 2 * m->ffn, H, H, TC_BM));
    SB_TRY(make_map(&o[4 * l + 3], m->w_down[l], H, m->ffn, m->ffn, TC_BM));
  }
  SB_TRY(make_map(&o[4 * m->n_layers], m->lm_head, m->vocab, H, H, TC_BM));
  return 0;
}

}  // namespace sb
