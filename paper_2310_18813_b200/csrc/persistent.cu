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
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "grid_sync.cuh"
#include "kernels.cuh"
#include "mma_ptx.cuh"
#include "tc_ptx.cuh"

namespace sb {

constexpr int PK_THREADS = 224;
constexpr int PK_MAX_T = 256;
constexpr int PK_MAX_G = 1024;
constexpr int PK_STAGE_PAD = 17;  // RoPE staging row stride (floats)

enum : int { PG_QKV = 0, PG_O = 1, PG_GU = 2, PG_DOWN = 3, PG_LM = 4 };
enum : int { PH_EMBED = 0, PH_GEMM = 1, PH_ATTN = 2, PH_FINAL = 3 };

struct PkGemm {
  int N, K, kb, n_tiles, units, ctas;
};

struct PkParams {
  int T, n_seq, q_len, H, nq, nkv, hd, ffn, V, L;
  int tn, G, n_phases, stages;
  int epi_bytes;
  int l2_ahead;  // units the L2 prefetch cursor runs ahead of the smem ring
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
  unsigned long long* trace;  // diagnostics: [G][n_phases][8] globaltimer ns (NULL = off)
};

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

// ------------------------------------------------------------------ work order
// Stream-K segments of CTA range [s, e) in PROCESSING order: the tail of a
// tile begun by another CTA ("contrib", published first so its owner never
// waits long), then the head of the tile this CTA owns (fix-up overlaps the
// MMA of the full tiles that follow), then whole tiles.
struct SegWalk {
  int kb, cs, ce, hs, he, fs, fe, k;
  __device__ __forceinline__ SegWalk(int s, int e, int kb_) : kb(kb_), cs(0), ce(0), hs(0), he(0), fs(0), fe(0), k(0) {
    if (s >= e) return;
    int f = s;
    if (s % kb) {
      cs = s;
      ce = min(e, (s / kb + 1) * kb);
      f = ce;
    }
    int fend = e;
    if (f < e && (e % kb)) {
      const int t1 = (e - 1) / kb * kb;
      if (t1 >= f) {
        hs = t1;
        he = e;
        fend = t1;
      }
    }
    if (f < fend) {
      fs = f;
      fe = fend;
    }
  }
  // next segment [a, b) of units; false when done
  __device__ __forceinline__ bool next(int& a, int& b) {
    if (k == 0) {
      k = 1;
      if (ce > cs) {
        a = cs;
        b = ce;
        return true;
      }
    }
    if (k == 1) {
      k = 2;
      if (he > hs) {
        a = hs;
        b = he;
        return true;
      }
    }
    if (fs < fe) {
      a = fs;
      b = fs + kb;
      fs = b;
      return true;
    }
    return false;
  }
};

// Attention work: item = (sequence, kv head, 16-query chunk); its keys
// [0, maxpos] stream through the shared TMA ring as "KV units" of UK keys
// (K and V tiles, 16 KB: UK = 32 at hd 128, 64 at hd 64).
struct AttnItem {
  int seq, kvh, chunk, n_units, maxp;
};
__device__ __forceinline__ AttnItem attn_item_of(const PkParams& p, int i) {
  AttnItem it;
  const int group = p.nq / p.nkv;
  const int nQ = group * p.q_len;
  const int n_chunks = (nQ + 15) / 16;
  it.chunk = i % n_chunks;
  it.kvh = (i / n_chunks) % p.nkv;
  it.seq = i / (n_chunks * p.nkv);
  int mp = -1;
  const int t0 = (it.chunk * 16) / group, t1 = min(nQ - 1, it.chunk * 16 + 15) / group;
  for (int t = t0; t <= t1; ++t) mp = max(mp, p.pos[it.seq * p.q_len + t]);
  it.maxp = mp;
  const int uk = 4096 / p.hd;
  it.n_units = (mp + 1 + uk - 1) / uk;
  return it;
}
__device__ __forceinline__ int attn_items(const PkParams& p) {
  const int group = p.nq / p.nkv;
  return p.n_seq * p.nkv * ((group * p.q_len + 15) / 16);
}
// row of the first key of unit v of an item in the [rows, hd] view of the cache
__device__ __forceinline__ int kv_row(const PkParams& p, int layer, const AttnItem& it, int v) {
  const int slot = p.slot[it.seq];
  return (int)((((size_t)layer * p.kv_slots + slot) * p.nkv + it.kvh) * p.ctx_max) + v * (4096 / p.hd);
}

// The CTA's ring work sequence (GEMM weight units and attention KV units, in
// ring order) as a resumable cursor: the weight producer walks it twice, once
// to fill the smem ring and once, `l2_ahead` units in front, to prefetch into L2.
struct UnitCursor {
  int ph, kind, layer, gk, a, b, u, i, v, nu, n_items;
  SegWalk sw;
  AttnItem item;
  __device__ __forceinline__ UnitCursor() : ph(0), kind(-1), layer(0), gk(0), a(0), b(0), u(0), i(0), v(0), nu(0),
                                            n_items(0), sw(0, 0, 1) {}
  // next unit; kind_out PH_GEMM (u_out = unit of gemm gk_out) or PH_ATTN (item_out, v_out)
  __device__ __forceinline__ bool next(const PkParams& p, int c, bool& waited, int& kind_out, int& layer_out,
                                       int& gk_out, int& u_out, AttnItem& item_out, int& v_out) {
    while (true) {
      if (kind == PH_GEMM) {
        if (u < b) {
          kind_out = PH_GEMM;
          layer_out = layer;
          gk_out = gk;
          u_out = u++;
          return true;
        }
        if (sw.next(a, b)) {
          u = a;
          continue;
        }
      } else if (kind == PH_ATTN) {
        if (v < nu) {
          kind_out = PH_ATTN;
          layer_out = layer;
          item_out = item;
          v_out = v++;
          return true;
        }
        i += p.G;
        if (i < n_items) {
          item = attn_item_of(p, i);
          nu = item.n_units;
          v = 0;
          continue;
        }
      }
      if (++ph >= p.n_phases) return false;
      kind = phase_kind(p, ph, layer, gk);
      if (kind == PH_GEMM) {
        int s, e;
        unit_range(p.g[gk], c, s, e);
        sw = SegWalk(s, e, p.g[gk].kb);
        u = b = 0;
      } else if (kind == PH_ATTN) {
        if (!waited) {
          griddep_wait();  // positions come from the previous kernel
          waited = true;
        }
        n_items = attn_items(p);
        i = c - p.G;
        v = nu = 0;
      } else {
        kind = -1;
      }
    }
  }
};

// swizzled (128B) smem address of 16-byte chunk `ch` (0..7) of row r in a
// [rows][128 B] TMA box; `base` 1024-aligned
__device__ __forceinline__ uint32_t sw_addr(uint32_t base, int r, int ch) {
  return base + (uint32_t)(r * 128) + (uint32_t)(((ch ^ (r & 7)) & 7) << 4);
}

// One warp's share (KW = 2048/HD keys) of one KV unit: S = Q K^T, online
// softmax, O += P V (mma.sync m16n8k16; Q fragments in registers).
template <int HD>
__device__ __forceinline__ void attn_unit(uint32_t kbase, uint32_t vbase, int key0, int kw, const uint32_t (&qa)[HD / 16][4],
                                          int pos_lo, int pos_hi, float scale, float (&o)[HD / 8][4], float& m_lo,
                                          float& m_hi, float& l_lo, float& l_hi) {
  constexpr int KSTEP = HD / 16, NT = HD / 8, UK = 4096 / HD, KW = UK / 2;
  const int lane = threadIdx.x & 31;
  const int mi = lane >> 3, ri = lane & 7;
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int sb = 0; sb < KW / 16; ++sb) {
    const int kl = kw + sb * 16;  // first key (within the unit) of this 16-key block
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const int key = kl + ri + (mi >> 1) * 8;
#pragma unroll
      for (int ks = 0; ks < KSTEP; ++ks) {
        const int col = ks * 16 + (mi & 1) * 8;  // element column
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sw_addr(kbase + (uint32_t)((col >> 6) * UK * 128), key, (col & 63) >> 3), b0, b1, b2, b3);
        mma_bf16(s0, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
        mma_bf16(s1, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
      }
    }
    const int kbase_i = key0 + kl + 2 * t4;
    float v[8] = {s0[0], s0[1], s1[0], s1[1], s0[2], s0[3], s1[2], s1[3]};
    const int kidx[4] = {kbase_i, kbase_i + 1, kbase_i + 8, kbase_i + 9};
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
      const int key = kl + ri + (mi & 1) * 8;
#pragma unroll
      for (int n = 0; n < NT; n += 2) {
        const int col = n * 8 + (mi >> 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sw_addr(vbase + (uint32_t)((col >> 6) * UK * 128), key, (col & 63) >> 3), b0, b1, b2, b3);
        mma_bf16(o[n], pa0, pa1, pa2, pa3, b0, b1);
        mma_bf16(o[n + 1], pa0, pa1, pa2, pa3, b2, b3);
      }
    }
  }
}

// The attention phase of one CTA: its items in order, KV units consumed from
// the ring by two warp pairs (pair q takes units q, q+2, ...; within a unit
// each warp takes half the keys), warps combined in order through smem.
template <int HD>
__device__ void attn_phase(const PkParams& p, const PkSmem& sm, uint32_t stage_bytes, int S, uint32_t& it, int c,
                           int* qpos, int* qtok, int* qhead) {
  constexpr int RS = HD + 8, KSTEP = HD / 16, NT = HD / 8, UK = 4096 / HD, KW = UK / 2;
  const int tid = threadIdx.x - 64, warp = tid >> 5, lane = tid & 31;
  const int pair = warp >> 1, wp = warp & 1;
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(sm.epi);
  float* comb = reinterpret_cast<float*>(sm.epi + (size_t)16 * RS * 2);
  float* cm = comb + 4 * 16 * HD;
  float* cl = cm + 4 * 16;
  const int group = p.nq / p.nkv;
  const int qd = p.nq * HD;
  const int G = p.G;
  const int n_items = attn_items(p);
  for (int i = c; i < n_items; i += G) {
    const AttnItem item = attn_item_of(p, i);
    if (tid < 16) {
      const int jj = item.chunk * 16 + tid;
      const int t = jj / group;
      const bool ok = jj < group * p.q_len;
      qtok[tid] = ok ? t : 0;
      qhead[tid] = item.kvh * group + (ok ? jj % group : 0);
      qpos[tid] = ok ? p.pos[item.seq * p.q_len + t] : -1;
    }
    epi_sync();
    for (int e = tid; e < 16 * (HD / 8); e += 128) {
      const int j = e / (HD / 8), cc = (e % (HD / 8)) * 8;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (qpos[j] >= 0)
        v = __ldcg(reinterpret_cast<const uint4*>(p.qr + (size_t)(item.seq * p.q_len + qtok[j]) * qd + qhead[j] * HD + cc));
      *reinterpret_cast<uint4*>(Qs + j * RS + cc) = v;
    }
    epi_sync();
    uint32_t qa[KSTEP][4];
    {
      const uint32_t qs_base = (uint32_t)__cvta_generic_to_shared(Qs);
      const int mi = lane >> 3, ri = lane & 7;
      const int r = ri + (mi & 1) * 8;
#pragma unroll
      for (int ks = 0; ks < KSTEP; ++ks)
        ldsm_x4(qs_base + (uint32_t)(r * RS + ks * 16 + (mi >> 1) * 8) * 2, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
    const int g = lane >> 2, t4 = lane & 3;
    const int pos_lo = qpos[g], pos_hi = qpos[g + 8];
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
    for (int v0 = 0; v0 < item.n_units; v0 += 2) {
      const int v = v0 + pair;
      if (v < item.n_units) {
        const uint32_t u = it + (uint32_t)v;
        const int stg = (int)(u % (uint32_t)S);
        mbar_wait(&sm.full[stg], (u / S) & 1);
        const uint32_t kb = smem_u32(sm.ring + (size_t)stg * stage_bytes);
        attn_unit<HD>(kb, kb + 8192, v * UK, wp * KW, qa, pos_lo, pos_hi, p.att_scale, o, m_lo, m_hi, l_lo, l_hi);
        asm volatile("bar.sync %0, 64;" ::"r"(2 + pair) : "memory");  // both warps of the pair are done with the stage
        if (wp == 0 && lane == 0) mbar_arrive(&sm.empty[stg]);
      }
      // lockstep: a pair may not run a ring's length ahead of the other (the
      // mbarrier parity of a stage two rounds ahead would alias)
      epi_sync();
    }
    it += (uint32_t)item.n_units;
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
      p.attn[((size_t)(item.seq * p.q_len + qtok[j]) * p.nq + qhead[j]) * HD + d] =
          __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
    }
    epi_sync();
  }
}

// ------------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(PK_THREADS, 1)
    persistent_forward_kernel(const __grid_constant__ CUtensorMap map_xb, const __grid_constant__ CUtensorMap map_attn,
                              const __grid_constant__ CUtensorMap map_act, const __grid_constant__ CUtensorMap map_lm,
                              const __grid_constant__ CUtensorMap map_kc, const __grid_constant__ CUtensorMap map_vc,
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
  off += p.epi_bytes;
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
  // attention phases finished by this CTA's epilogue warps: the MMA warp skips the
  // ring slots of KV units and must not run a ring round ahead of their consumers
  __shared__ int s_attn_done;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < 2 * tn) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    s_attn_done = 0;
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
  const uint32_t kv_unit_bytes = 16384;

  if (warp == 0) {
    // ================= weight producer: runs ahead through every GEMM phase
    // (weights depend neither on earlier phases nor on the previous kernel);
    // for the KV units of an attention phase it only arrives (the activation
    // producer loads them), keeping the ring's FIFO order.  A second cursor
    // `l2_ahead` units in front prefetches weights / KV into L2, so HBM keeps
    // streaming through phase tails and grid barriers.
    if (lane == 0) {
      uint32_t it = 0;
      bool waited = false;
      UnitCursor ld, pf;
      int kd, ly, gk, u, v;
      AttnItem item;
      auto prefetch = [&](int kd_, int ly_, int gk_, int u_, const AttnItem& item_, int v_) {
        if (kd_ == PH_GEMM) {
          const PkGemm& g = p.g[gk_];
          const int tile = u_ / g.kb, kbi = u_ - tile * g.kb;
          tma_prefetch_2d(wmap_of(p, ly_, gk_), kbi * TC_BK, tile * TC_BM);
        } else {
          const int r0 = kv_row(p, ly_, item_, v_);
          for (int h = 0; h < p.hd / 64; ++h) {
            tma_prefetch_2d(&map_kc, h * 64, r0);
            tma_prefetch_2d(&map_vc, h * 64, r0);
          }
        }
      };
      for (int k = 0; k < p.l2_ahead && pf.next(p, c, waited, kd, ly, gk, u, item, v); ++k)
        prefetch(kd, ly, gk, u, item, v);
      while (ld.next(p, c, waited, kd, ly, gk, u, item, v)) {
        {
          int kd2, ly2, gk2, u2, v2;
          AttnItem item2;
          if (p.l2_ahead > 0 && pf.next(p, c, waited, kd2, ly2, gk2, u2, item2, v2)) prefetch(kd2, ly2, gk2, u2, item2, v2);
        }
        const int stg = (int)(it % S);
        if (it >= (uint32_t)S) mbar_wait(&sm.empty[stg], ((it / S) + 1) & 1);
        if (kd == PH_ATTN) {
          mbar_arrive(&sm.full[stg]);
        } else {
          const PkGemm& g = p.g[gk];
          mbar_arrive_expect(&sm.full[stg], a_bytes);
          const int tile = u / g.kb, kbi = u - tile * g.kb;
          tma_load_2d(sm.ring + (size_t)stg * stage_bytes, wmap_of(p, ly, gk), &sm.full[stg], kbi * TC_BK, tile * TC_BM);
        }
        ++it;
      }
    }
  } else if (warp == 6) {
    // ================= activation producer: X tiles (and attention KV units)
    // of phase ph only after the grid barrier says every CTA finished phases < ph
    if (lane == 0) {
      griddep_wait();
      uint32_t it = 0;
      for (int ph = 1; ph < p.n_phases; ++ph) {
        int layer, gk;
        const int kind = phase_kind(p, ph, layer, gk);
        if (kind == PH_ATTN) {
          const int n_items = attn_items(p);
          if (c < n_items) {
            wait_geq(bar, (unsigned)(ph * G));
            fence_proxy_async();
          }
          for (int i = c; i < n_items; i += G) {
            const AttnItem item = attn_item_of(p, i);
            for (int v = 0; v < item.n_units; ++v, ++it) {
              const int stg = (int)(it % S);
              if (it >= (uint32_t)S) mbar_wait(&sm.empty[stg], ((it / S) + 1) & 1);
              mbar_arrive_expect(&sm.full[stg], kv_unit_bytes);
              const int r0 = kv_row(p, layer, item, v);
              uint8_t* dst = sm.ring + (size_t)stg * stage_bytes;
              const int uk = 4096 / p.hd;
              for (int h = 0; h < p.hd / 64; ++h) {
                tma_load_2d(dst + h * uk * 128, &map_kc, &sm.full[stg], h * 64, r0);
                tma_load_2d(dst + 8192 + h * uk * 128, &map_vc, &sm.full[stg], h * 64, r0);
              }
            }
          }
          continue;
        }
        if (kind != PH_GEMM) continue;
        const PkGemm& g = p.g[gk];
        const CUtensorMap* xm = gk == PG_O ? &map_attn : (gk == PG_DOWN ? &map_act : (gk == PG_LM ? &map_lm : &map_xb));
        int s, e;
        unit_range(g, c, s, e);
        if (s < e) {
          wait_geq(bar, (unsigned)(ph * G));
          fence_proxy_async();
        }
        SegWalk sw(s, e, g.kb);
        int a, b;
        while (sw.next(a, b)) {
          for (int u = a; u < b; ++u, ++it) {
            const int stg = (int)(it % S);
            if (it >= (uint32_t)S) mbar_wait(&sm.empty[stg], ((it / S) + 1) & 1);
            mbar_arrive_expect(&sm.full[stg], b_bytes);
            const int kbi = u % g.kb;
            tma_load_2d(sm.ring + (size_t)stg * stage_bytes + a_bytes, xm, &sm.full[stg], kbi * TC_BK, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (skips the ring slots of attention KV units)
    if (lane == 0) {
      const uint32_t idesc = make_idesc(tn);
      uint32_t it = 0, seg = 0;
      int n_attn = 0;
      bool waited = false;
      for (int ph = 1; ph < p.n_phases; ++ph) {
        int layer, gk;
        const int kind = phase_kind(p, ph, layer, gk);
        if (kind == PH_ATTN) {
          if (!waited) {
            griddep_wait();
            waited = true;
          }
          const int n_items = attn_items(p);
          for (int i = c; i < n_items; i += G) it += (uint32_t)attn_item_of(p, i).n_units;
          ++n_attn;
          while (*(volatile int*)&s_attn_done < n_attn) __nanosleep(20);
          continue;
        }
        if (kind != PH_GEMM) continue;
        const PkGemm& g = p.g[gk];
        int s, e;
        unit_range(g, c, s, e);
        SegWalk sw(s, e, g.kb);
        int a, b;
        while (sw.next(a, b)) {
          const int buf = seg & 1;
          const uint32_t use = seg >> 1;
          if (seg >= 2) mbar_wait(&sm.tempty[buf], (use + 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(buf * tn);
          for (int u = a; u < b; ++u, ++it) {
            const int stg = (int)(it % S);
            mbar_wait(&sm.full[stg], (it / S) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(sm.ring + (size_t)stg * stage_bytes);
            const uint32_t sb = sa + a_bytes;
#pragma unroll
            for (int kk = 0; kk < TC_BK / TC_UK; ++kk)
              tc_mma(d, sw128_desc(sa + kk * TC_UK * 2), sw128_desc(sb + kk * TC_UK * 2), idesc,
                     (u > a || kk > 0) ? 1u : 0u);
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
    uint32_t seg = 0, it = 0;
    for (int ph = 0; ph < p.n_phases; ++ph) {
      int layer, gk;
      const int kind = phase_kind(p, ph, layer, gk);
      unsigned long long* tr = p.trace ? p.trace + ((size_t)c * p.n_phases + ph) * 8 : nullptr;
      if (tr && et == 0) tr[0] = globaltimer();
      if (et == 0) wait_geq(bar, (unsigned)(ph * G));
      if (tr && et == 0) tr[1] = globaltimer();
      bool first_seg = true;
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
        if (p.hd == 128)
          attn_phase<128>(p, sm, stage_bytes, S, it, c, a_qpos, a_qtok, a_qhead);
        else
          attn_phase<64>(p, sm, stage_bytes, S, it, c, a_qpos, a_qtok, a_qhead);
        epi_sync();
        if (et == 0) *(volatile int*)&s_attn_done = layer + 1;
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
        it += (uint32_t)(e - s);
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
                for (int q0 = 0; q0 < P_in; q0 += 8) {  // 8 loads in flight, summed in order
                  float t8[8];
#pragma unroll
                  for (int i = 0; i < 8; ++i) t8[i] = q0 + i < P_in ? __ldcg(src + (size_t)(q0 + i) * T) : 0.f;
#pragma unroll
                  for (int i = 0; i < 8; ++i) sacc += t8[i];
                }
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
        SegWalk sw(s, e, g.kb);
        int a_u, b_u;
        while (sw.next(a_u, b_u)) {
          const int tile = a_u / g.kb;
          const int a0 = a_u - tile * g.kb;
          const int b1 = b_u - tile * g.kb;
          const bool contrib = a0 > 0;
          const bool owner = a0 == 0 && b1 < g.kb;
          const int buf = seg & 1;
          const uint32_t use = seg >> 1;
          const int n0 = tile * TC_BM;
          const int n = n0 + row;
          int c_last = c;
          if (owner) {
            while (c_last + 1 < g.ctas && unit_start(g, c_last + 1) < (tile + 1) * g.kb) ++c_last;
            if (et == 0) {
              if (tr) tr[4] = globaltimer();
              for (int c2 = c + 1; c2 <= c_last; ++c2) wait_geq(&flags[c2], (unsigned)(ph + 1));
              if (tr) tr[5] = globaltimer();
            }
          }
          mbar_wait(&sm.tfull[buf], use & 1);
          if (tr && et == 0 && first_seg) tr[2] = globaltimer();
          if (tr && et == 0) tr[6] = globaltimer();
          first_seg = false;
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
              // partial tile, row-major per weight row: [c][row][tn] (float4 stores / loads)
              float4* dst = reinterpret_cast<float4*>(p.scratch + ((size_t)c * TC_BM + row) * tn + j0);
#pragma unroll
              for (int q = 0; q < 4; ++q) __stcg(dst + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
              continue;
            }
            if (owner) {
              // contributors in CTA order, up to four partials in flight per batch
              for (int c0 = c + 1; c0 <= c_last; c0 += 4) {
                float4 pr[4][4];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                  if (c0 + w <= c_last) {
                    const float4* src =
                        reinterpret_cast<const float4*>(p.scratch + ((size_t)(c0 + w) * TC_BM + row) * tn + j0);
#pragma unroll
                    for (int q = 0; q < 4; ++q) pr[w][q] = __ldcg(src + q);
                  }
                }
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                  if (c0 + w <= c_last) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                      v[4 * q] += pr[w][q].x;
                      v[4 * q + 1] += pr[w][q].y;
                      v[4 * q + 2] += pr[w][q].z;
                      v[4 * q + 3] += pr[w][q].w;
                    }
                  }
                }
              }
            }
            if (gk == PG_QKV) {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = bf16r(v[j] * sm.inv_s[j0 + j]);
              const int rbase = region == 0 ? 0 : (region == 1 ? qd : qd + kd);
              const int d = (n - rbase) % p.hd;
              const int head = (n - rbase) / p.hd;
              __nv_bfloat16* kv_base = (region == 1 ? p.kc : p.vc) + (size_t)layer * p.layer_kv;
              if (region < 2) {
                const int half = p.hd >> 1;
#pragma unroll
                for (int j = 0; j < 16; ++j) stage_f[row * PK_STAGE_PAD + j] = v[j];
                epi_sync();
                const bool lo = d < half;
                const int prow = lo ? row + half : row - half;
                const int di = lo ? d : d - half;
                float cs[16], sn[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {  // table loads first, all in flight
                  const int ps = sm.s_pos[j0 + j];
                  const int pc = ps < 0 ? 0 : (ps >= p.max_pos ? p.max_pos - 1 : ps);
                  cs[j] = __ldg(&p.cosT[(size_t)pc * half + di]);
                  sn[j] = __ldg(&p.sinT[(size_t)pc * half + di]);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                  const int m = j0 + j;
                  if (m >= T || n >= N) continue;
                  const float xp = stage_f[prow * PK_STAGE_PAD + j];
                  const int ps = sm.s_pos[m];
                  const float r = lo ? v[j] * cs[j] - xp * sn[j] : v[j] * cs[j] + xp * sn[j];
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
              // all 16 residual loads in flight before any store (one L2 round trip per chunk)
              float rv[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int m = j0 + j;
                rv[j] = (m < T && n < N) ? __ldcg(&p.resid[(size_t)m * H + n]) : 0.f;
              }
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int m = j0 + j;
                float sq = 0.f;
                if (m < T && n < N) {
                  const size_t o = (size_t)m * H + n;
                  const float nv = rv[j] + v[j];
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
              if (tr) tr[7] = globaltimer();
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
          ++seg;
        }
      }
      // ---- phase done: publish (fence orders generic writes for other SMs' TMA reads)
      epi_sync();
      if (et == 0) {
        if (tr) tr[3] = globaltimer();
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
static int g_persistent = 0;  // sb_set_persistent (off by default: see DESIGN.md §4b)
static unsigned long long* g_pk_trace = nullptr;  // sb_debug_persistent_trace

// epilogue-warp smem region (phases use it one at a time): attention Q tile +
// 4-warp combine buffer, RoPE pair staging, per-quadrant norm / argmax partials
static size_t pk_epi_bytes(int hd, int tn) {
  size_t att = (size_t)16 * (hd + 8) * 2 + (size_t)4 * 16 * hd * 4 + 2 * 4 * 16 * 4;
  size_t e = att;
  if ((size_t)128 * PK_STAGE_PAD * 4 > e) e = (size_t)128 * PK_STAGE_PAD * 4;
  if ((size_t)8 * tn * 4 > e) e = (size_t)8 * tn * 4;
  return (e + 1023) & ~(size_t)1023;
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
  if (!g_persistent || m->arch != SB_ARCH_LLAMA || m->dtype != SB_BF16 || !m->tmaps || T > PK_MAX_T) return false;
  if (m->head_dim != 64 && m->head_dim != 128) return false;
  const int qd = m->n_heads * m->head_dim, kd = m->n_kv_heads * m->head_dim;
  if (qd % TC_BM || kd % TC_BM) return false;
  if (m->hidden % 8 || m->ffn % 8) return false;  // 16-byte TMA row strides
  if (m->n_heads % m->n_kv_heads) return false;
  return true;
}

#define PK_TRY(expr)                                                                           \
  do {                                                                                         \
    int rc_ = (expr);                                                                          \
    if (rc_ != 0) {                                                                            \
      if (getenv("SB_DEBUG")) fprintf(stderr, "persistent_forward: %s -> %d\n", #expr, rc_); \
      return rc_;                                                                              \
    }                                                                                          \
  } while (0)

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
  if (want_lm && !p.want_argmax && !p.want_logits) PK_TRY(SB_EINVAL);
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
  p.trace = g_pk_trace;
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
  p.epi_bytes = (int)epi;
  {
    static int ahead = -1;
    if (ahead < 0) {
      const char* env = getenv("SB_PK_L2_AHEAD");
      ahead = env ? atoi(env) : 0;  // measured: L2 prefetch ahead of the ring slows the stream
    }
    p.l2_ahead = ahead;
  }
  const size_t fixed = 1024 + epi + 3 * PK_MAX_T * 4 + 64 * 8 + 16;
  const size_t budget = 226 * 1024;
  const size_t stage = (size_t)(TC_BM + p.tn) * TC_BK * 2;
  int S = (int)((budget - fixed) / stage);
  if (S > 16) S = 16;
  if (S < 2) PK_TRY(SB_EUNSUPPORTED);
  p.stages = S;
  const size_t smem = 1024 + (size_t)S * stage + epi + 3 * PK_MAX_T * 4 + (2 * S + 4) * 8 + 16;
  static size_t attr_smem = 0;
  if (smem > attr_smem) {
    cudaError_t e = cudaFuncSetAttribute(persistent_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    PK_TRY((int)e);
    attr_smem = smem;
  }
  CUtensorMap mx, ma, mc, ml, mk, mv;
  {
    // KV cache as a 2-D [L*slots*nkv*ctx_max, hd] tensor: attention KV units of 4096/hd keys
    const int kv_rows = (int)((size_t)p.L * kv->slots * p.nkv * kv->ctx_max);
    PK_TRY(make_map(&mk, kv->k, kv_rows, p.hd, p.hd, 4096 / p.hd));
    PK_TRY(make_map(&mv, kv->v, kv_rows, p.hd, p.hd, 4096 / p.hd));
  }
  PK_TRY(make_map(&mx, b.xb, T, p.H, p.H, p.tn));
  PK_TRY(make_map(&ma, b.attn, T, qd, qd, p.tn));
  PK_TRY(make_map(&mc, b.act, T, p.ffn, p.ffn, p.tn));
  if (want_lm) {
    PK_TRY(make_map(&ml, (const char*)b.xb + (size_t)p.lm_off * p.H * 2, p.lm_rows, p.H, p.lm_step * p.H, p.tn));
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, persistent_forward_kernel, mx, ma, mc, ml, mk, mv, p);
  if (e != cudaSuccess) {
    fprintf(stderr, "specbatch_b200: persistent forward launch failed: %s (T=%d tn=%d stages=%d smem=%zu)\n",
            cudaGetErrorString(e), T, p.tn, S, smem);
    return (int)e;
  }
  ++g_kernel_count;
  return 0;
}

int set_persistent_trace(void* buf) {
  g_pk_trace = (unsigned long long*)buf;
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
