// K1: the whole greedy draft loop of one speculative iteration -- k autoregressive
// steps of the small Llama draft for b sequences -- in ONE persistent launch.
//
// Reference: the draft proposals of DraftOracle.step / TokenLevel.draft_tokens
// (engine.py:100-106, 138-145), charged k * ssm_step_time per iteration
// (engine.py:196-198).  The per-step path issues ~13 dependent kernels per draft
// step; each pays launch + prologue latency while the 68M draft's weights are
// only ~87 MB (13 us of HBM, ~7 us of L2).  Here one CTA per SM runs every step:
//
//   per step j: [embed + 1/rms of the step's tokens, rebuilt in every CTA]
//     per layer:  A qkv (fused 1/rms, RoPE, KV append) | B attention | C o (+resid)
//                 | D gate/up (silu*up) | E down (+resid, 4-CTA cluster split-K)
//     F lm_head (fused 1/rms, per-CTA argmax partials) | G argmax -> next tokens
//
// separated by grid barriers (sense-free monotonic counter, one red.release per
// CTA, one polling thread).  The weight stream is DECOUPLED from the barriers: a
// producer warp walks this CTA's tile schedule for the whole launch and keeps a
// ring of NS shared-memory slots full with 1-D bulk copies (16 weight rows x K
// per tile, L2 evict-last: the draft is re-read every step), so the next phase's
// weights are already on chip while the grid waits at a barrier.  The eight
// consumer warps split each tile's K over warps (mma.sync m16n8k16, bf16 in /
// fp32 accumulate; tokens are the N dimension, T <= 16), reduce through shared
// memory in fixed warp order and run the phase epilogue; the down projection's
// K = ffn is split over the 4 CTAs of a thread-block cluster and reduced in rank
// order through DSMEM (deterministic, no global fix-up).
//
// Outputs follow the token-sink protocol of sb_decoder_forward_ex:
//   v_ids[s*(k+1) + j] = d_j,  ds_ids[s] = d_j,  ds_pos[s] = d_base[s] + j.
// Numerics follow the engine's fused-norm contract: GEMM inputs are
// bf16(residual * gain), outputs scaled by 1/rms(residual); residual fp32.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "mma_ptx.cuh"
#include "tc_ptx.cuh"

namespace sb {

namespace dl {

constexpr int kThreads = 288;  // 8 consumer warps + 1 producer warp
constexpr int kConsumers = 256;
constexpr int kMaxT = 16;      // tokens per step (2b in step 1)
constexpr int kMaxB = 8;
constexpr int kMaxL = 16;
constexpr int kHd = 64;        // head_dim (RoPE pairs d, d+32 live in one 16-row tile)
constexpr int kMaxCS = 8;

struct Params {
  int L, H, nq, nkv, ffn, V, max_pos, ctx_max, slots, b, k, G, CS, NS;
  float eps, att_scale;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* lm_head;
  const __nv_bfloat16* final_norm;
  const __nv_bfloat16* attn_norm[kMaxL];
  const __nv_bfloat16* mlp_norm[kMaxL];
  const __nv_bfloat16* w_qkv[kMaxL];
  const __nv_bfloat16* w_o[kMaxL];
  const __nv_bfloat16* w_gu[kMaxL];
  const __nv_bfloat16* w_down[kMaxL];
  const float* cosT;
  const float* sinT;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  size_t layer_kv;  // elements per layer of one cache (slots * nkv * ctx_max * hd)
  const int32_t* d1_ids;
  const int32_t* d1_pos;
  const int32_t* slot;
  const int32_t* d_base;
  int32_t* v_ids;
  int32_t* ds_ids;
  int32_t* ds_pos;
  float* resid;          // [kMaxT][H]
  __nv_bfloat16* xb;     // [kMaxT][H]   bf16(resid * next gain)
  __nv_bfloat16* qr;     // [kMaxT][H]   rotated q
  __nv_bfloat16* attn;   // [kMaxT][H]
  __nv_bfloat16* act;    // [kMaxT][ffn]
  float* npart;          // [H/16][kMaxT] sum of squares of the new residual per 16-column unit
  float* am_val;         // [G][kMaxB]
  int* am_idx;
  unsigned long long* bar_count;  // grid barrier (self-resetting)
  unsigned* exit_count;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void named_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ------------------------------------------------------------------ tile schedule
// Phases with weight tiles (16 rows x H of K each): A qkv, C o, D gate/up, E down
// (16 rows x one H-wide K chunk; chunk = cluster rank), F lm_head.  Tiles of
// A/C/D/F go round-robin over the G CTAs with a per-phase rotation (t + off) % G;
// E: cluster q takes units q, q + NCL, ... and rank r its r-th K chunk.
struct Sched {
  int G, c, nA, nC, nD, nE, nF, NCL, cid, rank;
  __device__ int offA() const { return 0; }
  __device__ int offC() const { return nA % G; }
  __device__ int offD() const { return (nA + nC) % G; }
  __device__ int offF() const { return (nA + nC + nD) % G; }
  // first tile of this CTA in a phase with n tiles and rotation off (tiles: first, first + G, ...)
  __device__ int first(int off) const { return (c - off + G) % G; }
};

// qkv tile u -> weight row of its r-th row (RoPE pairs (d, d+32) in rows r, r+8)
__device__ __forceinline__ int qkv_row(int u, int r) {
  const int hs = u >> 2, j = u & 3;
  return hs * kHd + (r < 8 ? 8 * j + r : 32 + 8 * j + (r - 8));
}

// ------------------------------------------------------------------ producer
__device__ void producer(const Params& p, const Sched& S, uint8_t* ring, uint64_t* full, uint64_t* empty, int srow) {
  const uint64_t pol = l2_policy_evict_last();
  const uint32_t rowb = (uint32_t)p.H * 2;
  int n = 0;
  auto put = [&](const __nv_bfloat16* base, size_t row_stride, auto row_of) {
    const int s = n % p.NS;
    if (n >= p.NS) mbar_wait(&empty[s], ((n / p.NS) + 1) & 1);
    mbar_expect_tx(&full[s], 16 * rowb);
    uint8_t* dst = ring + (size_t)s * 16 * srow;
#pragma unroll 1
    for (int r = 0; r < 16; ++r) bulk_g2s(dst + r * srow, base + (size_t)row_of(r) * row_stride, rowb, &full[s], pol);
    ++n;
  };
  for (int j = 0; j < p.k; ++j) {
    for (int l = 0; l < p.L; ++l) {
      for (int u = S.first(S.offA()); u < S.nA; u += S.G) put(p.w_qkv[l], p.H, [&](int r) { return qkv_row(u, r); });
      for (int u = S.first(S.offC()); u < S.nC; u += S.G) put(p.w_o[l], p.H, [&](int r) { return 16 * u + r; });
      for (int u = S.first(S.offD()); u < S.nD; u += S.G) put(p.w_gu[l], p.H, [&](int r) { return 16 * u + r; });
      for (int u = S.cid; u < S.nE; u += S.NCL)
        if (S.rank < p.CS) put(p.w_down[l] + (size_t)S.rank * p.H, p.ffn, [&](int r) { return 16 * u + r; });
    }
    for (int u = S.first(S.offF()); u < S.nF; u += S.G) put(p.lm_head, p.H, [&](int r) { return 16 * u + r; });
  }
}

// ------------------------------------------------------------------ consumer pieces
struct Smem {
  uint8_t* ring;
  __nv_bfloat16* xs;  // [kMaxT][H + 8]
  float* red;         // [2][8 warps][kMaxT][16]
  float* dpart;       // [2 rounds][kMaxCS][kMaxT][16]   (cluster leader)
  float* qs;          // [2][kHd] attention queries
  float* att;         // [8 warps][2][kHd + 2]  attention partials (o, m, l)
  float* rinv;        // [kMaxT]
  int* tid_tok;       // [kMaxT] token ids of the step
  int* tpos;          // [kMaxT] positions
  int* tok_next;      // [kMaxB]
  uint64_t* full;
  uint64_t* empty;
  uint64_t* ebar;     // [2] cluster-reduce barriers (leader)
  int srow, xrow;
};

// grid barrier #idx (0-based over the launch): all G CTAs' consumer threads
__device__ __forceinline__ void grid_bar(const Params& p, int& nbar) {
  named_bar();
  ++nbar;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p.bar_count) : "memory");
    const unsigned long long target = (unsigned long long)nbar * p.G;
    if (ld_acquire_u64(p.bar_count) < target) {
      uint64_t t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while (ld_acquire_u64(p.bar_count) < target) {
        uint64_t t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 2000000000ull) __trap();  // 2 s: a co-residency / protocol bug errors out instead of hanging
      }
    }
  }
  named_bar();
}

// X staging: rows t < T of src (row stride ld elements, first element col0) -> xs
__device__ __forceinline__ void load_x(const Smem& sm, const __nv_bfloat16* src, int ld, int T, int H,
                                       int row_step = 1, int row_off = 0) {
  const int vec = H / 8;
  for (int e = threadIdx.x; e < T * vec; e += kConsumers) {
    const int t = e / vec, v = e % vec;
    cp_async16(sm.xs + (size_t)t * sm.xrow + v * 8, src + (size_t)(t * row_step + row_off) * ld + v * 8);
  }
  cp_async_commit();
  cp_async_wait<0>();
}

// 1/rms per token from the producer partials npart[unit][t] (n units, fixed order)
__device__ __forceinline__ void load_rinv(const Smem& sm, const Params& p, int T, int row_step = 1, int row_off = 0) {
  const int nU = p.H / 16;
  if ((int)threadIdx.x < T) {
    const int t = threadIdx.x * row_step + row_off;
    float ss = 0.f;
    for (int u = 0; u < nU; ++u) ss += __ldcg(p.npart + u * kMaxT + t);
    sm.rinv[threadIdx.x] = rsqrtf(ss / (float)p.H + p.eps);
  }
}

// One tile: wait for slot, split-K mma over the 8 consumer warps, partials -> red[buf],
// barrier, release the slot.  Returns the reduced value of (row r = tid & 15, token t = tid >> 4).
__device__ __forceinline__ float tile_mma(const Smem& sm, int H, int NS, int& n, int T) {
  const int s = n % NS;
  mbar_wait(&sm.full[s], (n / NS) & 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ksteps = H / 16, per = (ksteps + 7) / 8;
  const int k0 = warp * per, k1 = min(ksteps, k0 + per);
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  const uint32_t wa = smem_u32(sm.ring + (size_t)s * 16 * sm.srow) + (uint32_t)((lane & 15) * sm.srow + (lane >> 4) * 16);
  const int tok = (lane & 7) + (lane >> 4) * 8;
  const uint32_t xa = smem_u32(sm.xs) + (uint32_t)((tok * sm.xrow + ((lane >> 3) & 1) * 8) * 2);
  const bool two = T > 8;
  for (int kk = k0; kk < k1; ++kk) {
    uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
    ldsm_x4(wa + kk * 32, a0, a1, a2, a3);
    ldsm_x4(xa + kk * 32, b0, b1, b2, b3);
    mma_bf16(acc[0], a0, a1, a2, a3, b0, b1);
    if (two) mma_bf16(acc[1], a0, a1, a2, a3, b2, b3);
  }
  const int buf = n & 1;
  float* red = sm.red + (size_t)(buf * 8 + warp) * kMaxT * 16;
  const int row = lane >> 2, tc = (lane & 3) * 2;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    red[(nt * 8 + tc) * 16 + row] = acc[nt][0];
    red[(nt * 8 + tc + 1) * 16 + row] = acc[nt][1];
    red[(nt * 8 + tc) * 16 + row + 8] = acc[nt][2];
    red[(nt * 8 + tc + 1) * 16 + row + 8] = acc[nt][3];
  }
  named_bar();
  if (threadIdx.x == 0) mbar_arrive(&sm.empty[s]);
  ++n;
  const float* rb = sm.red + (size_t)buf * 8 * kMaxT * 16 + threadIdx.x;
  float v = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) v += rb[w * kMaxT * 16];
  return v;
}

__device__ __forceinline__ float silu(float g) { return g / (1.f + __expf(-g)); }

// Residual epilogue (o_proj / down_proj): resid[t][16u + r] += v; xb = bf16(new * gain); npart[u][t]
__device__ __forceinline__ void resid_epilogue(const Params& p, float v, int u, int T, const __nv_bfloat16* gain) {
  const int r = threadIdx.x & 15, t = threadIdx.x >> 4;
  float sq = 0.f;
  if (t < T) {
    const size_t o = (size_t)t * p.H + 16 * u + r;
    const float nv = __ldcg(p.resid + o) + v;
    __stcg(p.resid + o, nv);
    p.xb[o] = __float2bfloat16_rn(nv * __bfloat162float(gain[16 * u + r]));
    sq = nv * nv;
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (r == 0 && t < T) __stcg(p.npart + u * kMaxT + t, sq);
}

// Attention over the slot's cache for one (q head, sequence): q_len <= 2 queries, keys [0, pos].
__device__ void attention_unit(const Params& p, const Smem& sm, int l, int h, int s, int q, const __nv_bfloat16* kc,
                               const __nv_bfloat16* vc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = s * q;
  const int hk = h / (p.nq / p.nkv);
  const int slot = p.slot[s];
  for (int e = threadIdx.x; e < q * kHd; e += kConsumers) {
    const int i = e / kHd, d = e % kHd;
    sm.qs[i * kHd + d] = __bfloat162float(__ushort_as_bfloat16(__ldcg(reinterpret_cast<const unsigned short*>(p.qr) + (size_t)(t0 + i) * p.H + h * kHd + d)));
  }
  named_bar();
  int pos_i[2] = {sm.tpos[t0], sm.tpos[t0 + q - 1]};
  const int n_keys = pos_i[1] + 1;
  const int per = (n_keys + 7) / 8;
  const int kb = warp * per, ke = min(n_keys, kb + per);
  const size_t slab = ((size_t)slot * p.nkv + hk) * p.ctx_max * kHd;
  const __nv_bfloat16* K = kc + slab;
  const __nv_bfloat16* Vv = vc + slab;
  float m[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f}, o0[2] = {0.f, 0.f}, o1[2] = {0.f, 0.f};
  for (int base = kb; base < ke; base += 32) {
    const int key = base + lane;
    const bool ok = key < ke;
    float sc[2] = {-INFINITY, -INFINITY};
    if (ok) {
      const uint4* kr = reinterpret_cast<const uint4*>(K + (size_t)key * kHd);
      float d0 = 0.f, d1 = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 w = __ldcg(kr + c);
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(hv[e]);
          const int d = c * 8 + e * 2;
          d0 += f.x * sm.qs[d] + f.y * sm.qs[d + 1];
          if (q > 1) d1 += f.x * sm.qs[kHd + d] + f.y * sm.qs[kHd + d + 1];
        }
      }
      if (key <= pos_i[0]) sc[0] = d0 * p.att_scale;
      if (q > 1 && key <= pos_i[1]) sc[1] = d1 * p.att_scale;
    }
    float pr[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float cm = warp_max(sc[i]);
      const float nm = fmaxf(m[i], cm);
      const float corr = nm == -INFINITY ? 1.f : __expf(m[i] - nm);
      pr[i] = sc[i] == -INFINITY ? 0.f : __expf(sc[i] - nm);
      lsum[i] = lsum[i] * corr + warp_sum(pr[i]);
      o0[i] *= corr;
      o1[i] *= corr;
      m[i] = nm;
    }
    const int nk = min(32, ke - base);
    for (int kk = 0; kk < nk; ++kk) {
      const __nv_bfloat162 vv = __ldcg(reinterpret_cast<const __nv_bfloat162*>(Vv + (size_t)(base + kk) * kHd) + lane);
      const float2 vf = __bfloat1622float2(vv);
      const float p0 = __shfl_sync(0xffffffffu, pr[0], kk);
      const float p1 = __shfl_sync(0xffffffffu, pr[1], kk);
      o0[0] += p0 * vf.x;
      o1[0] += p0 * vf.y;
      o0[1] += p1 * vf.x;
      o1[1] += p1 * vf.y;
    }
  }
  float* aw = sm.att + (size_t)warp * 2 * (kHd + 2);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    aw[i * (kHd + 2) + 2 * lane] = o0[i];
    aw[i * (kHd + 2) + 2 * lane + 1] = o1[i];
    if (lane == 0) {
      aw[i * (kHd + 2) + kHd] = m[i];
      aw[i * (kHd + 2) + kHd + 1] = lsum[i];
    }
  }
  named_bar();
  if ((int)threadIdx.x < q * kHd) {
    const int i = threadIdx.x / kHd, d = threadIdx.x % kHd;
    float M = -INFINITY;
    for (int w = 0; w < 8; ++w) M = fmaxf(M, sm.att[(w * 2 + i) * (kHd + 2) + kHd]);
    float Ls = 0.f, O = 0.f;
    for (int w = 0; w < 8; ++w) {
      const float* a = sm.att + (w * 2 + i) * (kHd + 2);
      const float sc = a[kHd] == -INFINITY ? 0.f : __expf(a[kHd] - M);
      Ls += a[kHd + 1] * sc;
      O += a[d] * sc;
    }
    p.attn[(size_t)(t0 + i) * p.H + h * kHd + d] = __float2bfloat16_rn(Ls > 0.f ? O / Ls : 0.f);
  }
  named_bar();
}

// step inputs: token ids / positions -> embedding (+ attn_norm[0] gain) in xs, 1/rms, residual columns
__device__ void embed_step(const Params& p, const Smem& sm, int c, int T) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const __nv_bfloat16* g = p.attn_norm[0];
  for (int t = warp; t < T; t += 8) {
    const int id = sm.tid_tok[t];
    const bool pad = sm.tpos[t] < 0 || id < 0 || id >= p.V;
    const __nv_bfloat16* row = p.embed + (size_t)(pad ? 0 : id) * p.H;
    float ss = 0.f;
    for (int i = lane * 8; i < p.H; i += 256) {
      const uint4 w = pad ? make_uint4(0, 0, 0, 0) : __ldg(reinterpret_cast<const uint4*>(row + i));
      const uint4 gw = __ldg(reinterpret_cast<const uint4*>(g + i));
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&w);
      const __nv_bfloat162* gv = reinterpret_cast<const __nv_bfloat162*>(&gw);
      uint4 outw;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&outw);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(hv[e]);
        const float2 gf = __bfloat1622float2(gv[e]);
        ss += f.x * f.x + f.y * f.y;
        ow[e] = pack_bf16(f.x * gf.x, f.y * gf.y);
      }
      *reinterpret_cast<uint4*>(sm.xs + (size_t)t * sm.xrow + i) = outw;
    }
    ss = warp_sum(ss);
    if (lane == 0) sm.rinv[t] = rsqrtf(ss / (float)p.H + p.eps);
  }
  // the fp32 residual (the embedding) of columns [16c, 16c + 16): read-modified by the o / down owners
  if (c < p.H / 16) {
    for (int e = threadIdx.x; e < T * 16; e += kConsumers) {
      const int t = e >> 4, col = 16 * c + (e & 15);
      const int id = sm.tid_tok[t];
      const bool pad = sm.tpos[t] < 0 || id < 0 || id >= p.V;
      __stcg(p.resid + (size_t)t * p.H + col, pad ? 0.f : __bfloat162float(p.embed[(size_t)id * p.H + col]));
    }
  }
  named_bar();
}

__global__ void __launch_bounds__(kThreads, 1) draft_loop_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int H = p.H;
  Smem sm;
  sm.srow = H * 2 + 16;
  sm.xrow = H + 8;
  uint8_t* q = smem_raw;
  sm.ring = q;
  q += (size_t)p.NS * 16 * sm.srow;
  sm.xs = reinterpret_cast<__nv_bfloat16*>(q);
  q += (size_t)kMaxT * sm.xrow * 2;
  sm.red = reinterpret_cast<float*>(q);
  q += 2 * 8 * kMaxT * 16 * 4;
  sm.dpart = reinterpret_cast<float*>(q);
  q += 2 * kMaxCS * kMaxT * 16 * 4;
  sm.qs = reinterpret_cast<float*>(q);
  q += 2 * kHd * 4;
  sm.att = reinterpret_cast<float*>(q);
  q += 8 * 2 * (kHd + 2) * 4;
  sm.rinv = reinterpret_cast<float*>(q);
  q += kMaxT * 4;
  sm.tid_tok = reinterpret_cast<int*>(q);
  q += kMaxT * 4;
  sm.tpos = reinterpret_cast<int*>(q);
  q += kMaxT * 4;
  sm.tok_next = reinterpret_cast<int*>(q);
  q += kMaxB * 4;
  q = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(q) + 7) & ~uintptr_t(7));
  sm.full = reinterpret_cast<uint64_t*>(q);
  sm.empty = sm.full + p.NS;
  sm.ebar = sm.empty + p.NS;

  Sched S;
  S.G = p.G;
  S.c = blockIdx.x;
  S.nA = (p.nq + 2 * p.nkv) * kHd / 16;
  S.nC = H / 16;
  S.nD = 2 * p.ffn / 16;
  S.nE = H / 16;
  S.nF = p.V / 16;
  S.NCL = p.G / p.CS;
  S.cid = cluster_id();
  S.rank = cluster_rank();

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.NS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.ebar[0], p.CS - 1);
    mbar_init(&sm.ebar[1], p.CS - 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();  // barriers initialised before any remote arrive

  if (threadIdx.x >= kConsumers) {
    if (threadIdx.x == kConsumers) producer(p, S, sm.ring, sm.full, sm.empty, sm.srow);  // weights: no dependency
    return;
  }
  griddep_wait();  // committed tokens / staging written by the previous kernels
  const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = p.b;
  int n = 0, nbar = 0;
  int e_use[2] = {0, 0};
  float am_v = -INFINITY;  // running argmax (lm_head) of token t = tid >> 4 (held by r == 0 lanes)
  int am_i = 0;
  for (int j = 1; j <= p.k; ++j) {
    const int qn = j == 1 ? 2 : 1;
    const int T = b * qn;
    if (tid < T) {
      const int s = tid / qn;
      if (j == 1) {
        sm.tid_tok[tid] = p.d1_ids[tid];
        sm.tpos[tid] = p.d1_pos[tid];
      } else {
        sm.tid_tok[tid] = sm.tok_next[s];
        sm.tpos[tid] = p.d_base[s] + j - 1;
      }
    }
    named_bar();
    embed_step(p, sm, c, T);
    for (int l = 0; l < p.L; ++l) {
      const __nv_bfloat16* kcl = p.kc + (size_t)l * p.layer_kv;
      const __nv_bfloat16* vcl = p.vc + (size_t)l * p.layer_kv;
      // ---- A: qkv + 1/rms + RoPE + KV append
      if (l > 0 && S.first(S.offA()) < S.nA) {
        load_x(sm, p.xb, H, T, H);
        load_rinv(sm, p, T);
        named_bar();
      }
      for (int u = S.first(S.offA()); u < S.nA; u += S.G) {
        const float acc = tile_mma(sm, H, p.NS, n, T);
        const int r = tid & 15, t = tid >> 4;
        const float v = t < T ? __bfloat162float(__float2bfloat16_rn(acc * sm.rinv[t])) : 0.f;
        const float partner = __shfl_xor_sync(0xffffffffu, v, 8);
        const int hs = u >> 2, jj = u & 3;
        const int i = 8 * jj + (r & 7);  // rotary pair index (dims i, i + 32)
        if (t < T) {
          const int pos = sm.tpos[t];
          const int pc = pos < 0 ? 0 : (pos >= p.max_pos ? p.max_pos - 1 : pos);
          const int d = qkv_row(u, r) - hs * kHd;
          float out = v;
          if (hs < p.nq + p.nkv) {  // q or k: rotate-half
            const float cs = p.cosT[(size_t)pc * (kHd / 2) + i], sn = p.sinT[(size_t)pc * (kHd / 2) + i];
            out = r < 8 ? v * cs - partner * sn : v * cs + partner * sn;
          }
          const __nv_bfloat16 ob = __float2bfloat16_rn(out);
          if (hs < p.nq) {
            p.qr[(size_t)t * H + hs * kHd + d] = ob;
          } else if (pos >= 0) {
            const int s = t / qn;
            const int kvh = hs < p.nq + p.nkv ? hs - p.nq : hs - p.nq - p.nkv;
            __nv_bfloat16* dst = (hs < p.nq + p.nkv ? p.kc : p.vc) + (size_t)l * p.layer_kv +
                                 (((size_t)p.slot[s] * p.nkv + kvh) * p.ctx_max + pos) * kHd + d;
            *dst = ob;
          }
        }
      }
      grid_bar(p, nbar);
      // ---- B: attention (causal inside the window)
      for (int un = c; un < p.nq * b; un += S.G) attention_unit(p, sm, l, un % p.nq, un / p.nq, qn, kcl, vcl);
      grid_bar(p, nbar);
      // ---- C: o_proj (+ residual, bf16 copy * mlp gain, norm partials)
      if (S.first(S.offC()) < S.nC) {
        load_x(sm, p.attn, H, T, H);
        named_bar();
      }
      for (int u = S.first(S.offC()); u < S.nC; u += S.G) {
        const float acc = tile_mma(sm, H, p.NS, n, T);
        resid_epilogue(p, acc, u, T, p.mlp_norm[l]);
      }
      grid_bar(p, nbar);
      // ---- D: gate/up (interleaved rows) -> silu(g) * u
      if (S.first(S.offD()) < S.nD) {
        load_x(sm, p.xb, H, T, H);
        load_rinv(sm, p, T);
        named_bar();
      }
      for (int u = S.first(S.offD()); u < S.nD; u += S.G) {
        const float acc = tile_mma(sm, H, p.NS, n, T);
        const int r = tid & 15, t = tid >> 4;
        const float v = t < T ? acc * sm.rinv[t] : 0.f;
        const float up = __shfl_xor_sync(0xffffffffu, v, 1);
        if (t < T && !(r & 1)) p.act[(size_t)t * p.ffn + 8 * u + (r >> 1)] = __float2bfloat16_rn(silu(v) * up);
      }
      grid_bar(p, nbar);
      // ---- E: down_proj, K split over the cluster ranks, reduced in rank order at rank 0
      if (S.cid < S.nE && S.rank < p.CS) {
        load_x(sm, p.act + (size_t)S.rank * H, p.ffn, T, H);
        named_bar();
      }
      {
        const __nv_bfloat16* gnext = l + 1 < p.L ? p.attn_norm[l + 1] : p.final_norm;
        int round = 0;
        for (int u = S.cid; u < S.nE; u += S.NCL, ++round) {
          const float acc = tile_mma(sm, H, p.NS, n, T);
          const int rb = round & 1;
          float* dp = sm.dpart + (size_t)rb * kMaxCS * kMaxT * 16;
          if (S.rank == 0) {
            dp[tid] = acc;
            mbar_wait_cluster(&sm.ebar[rb], e_use[rb] & 1);
            ++e_use[rb];
            float v = 0.f;
            for (int r = 0; r < p.CS; ++r) v += dp[r * kMaxT * 16 + tid];
            resid_epilogue(p, v, u, T, gnext);
          } else {
            st_cluster_f32(map_rank(smem_u32(dp + S.rank * kMaxT * 16 + tid), 0), acc);
            named_bar();
            if (tid == 0) mbar_arrive_remote(map_rank(smem_u32(&sm.ebar[rb]), 0));
          }
        }
      }
      grid_bar(p, nbar);
    }
    // ---- F: lm_head over the last token of each sequence, fused 1/rms + argmax partials
    if (S.first(S.offF()) < S.nF) {
      load_x(sm, p.xb, H, b, H, qn, qn - 1);
      load_rinv(sm, p, b, qn, qn - 1);
      named_bar();
    }
    am_v = -INFINITY;
    am_i = 0;
    for (int u = S.first(S.offF()); u < S.nF; u += S.G) {
      const float acc = tile_mma(sm, H, p.NS, n, b);
      const int r = tid & 15, t = tid >> 4;
      ArgMax a{t < b ? acc * sm.rinv[t] : -INFINITY, 16 * u + r};
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        ArgMax x{__shfl_xor_sync(0xffffffffu, a.v, o), __shfl_xor_sync(0xffffffffu, a.i, o)};
        a = argmax_merge(a, x);
      }
      if (r == 0) {
        const ArgMax cur = argmax_merge(ArgMax{am_v, am_i}, a);
        am_v = cur.v;
        am_i = cur.i;
      }
    }
    if ((tid & 15) == 0 && (tid >> 4) < b) {
      __stcg(p.am_val + c * kMaxB + (tid >> 4), am_v);
      __stcg(p.am_idx + c * kMaxB + (tid >> 4), am_i);
    }
    grid_bar(p, nbar);
    // ---- G: argmax over the CTA partials -> d_j (every CTA: the next step's tokens)
    if (warp < b) {
      ArgMax a{-INFINITY, INT_MAX};
      for (int cc = lane; cc < S.G; cc += 32) {
        const float v = __ldcg(p.am_val + cc * kMaxB + warp);
        if (v == -INFINITY) continue;  // a CTA without lm_head tiles
        a = argmax_merge(a, ArgMax{v, __ldcg(p.am_idx + cc * kMaxB + warp)});
      }
      a = warp_argmax(a);
      if (lane == 0) {
        sm.tok_next[warp] = a.i;
        if (c == 0) {
          p.v_ids[warp * (p.k + 1) + j] = a.i;
          p.ds_ids[warp] = a.i;
          p.ds_pos[warp] = p.d_base[warp] + j;
        }
      }
    }
    named_bar();
  }
  griddep_launch();
  // self-reset of the barrier words for the next launch (every CTA has passed its last poll)
  if (tid == 0) {
    const unsigned old = atomicAdd(p.exit_count, 1u);
    if (old == (unsigned)p.G - 1) {
      atomicExch(p.bar_count, 0ull);
      atomicExch(p.exit_count, 0u);
    }
  }
}

}  // namespace dl

static int g_dl_enabled = 1;
static int g_dl_clusters[9] = {0};  // max co-resident clusters per cluster size (1 CTA per SM)

static size_t dl_smem_bytes(int H, int NS) {
  size_t b = (size_t)NS * 16 * (H * 2 + 16) + (size_t)dl::kMaxT * (H + 8) * 2 + 2 * 8 * dl::kMaxT * 16 * 4 +
             2 * dl::kMaxCS * dl::kMaxT * 16 * 4 + 2 * dl::kHd * 4 + 8 * 2 * (dl::kHd + 2) * 4 + 3 * dl::kMaxT * 4 +
             dl::kMaxB * 4 + 16;
  return b + (size_t)(2 * NS + 2) * 8;
}
constexpr size_t kDlSmemMax = 227 * 1024;

int draft_loop_init() {
  cudaError_t e = cudaFuncSetAttribute(dl::draft_loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDlSmemMax);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(dl::draft_loop_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return (int)e;
  for (int cs = 2; cs <= 8; cs *= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(dl::kThreads);
    cfg.dynamicSmemBytes = kDlSmemMax;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, dl::draft_loop_kernel, &cfg);
    if (e != cudaSuccess) return (int)e;
    g_dl_clusters[cs] = ncl;
  }
  return 0;
}

int draft_loop_grid(int cs) { return (cs >= 2 && cs <= 8) ? g_dl_clusters[cs] * cs : 0; }

}  // namespace sb

using namespace sb;

extern "C" {

int sb_set_draft_loop(int32_t enabled) {
  g_dl_enabled = enabled ? 1 : 0;
  return 0;
}

size_t sb_draft_loop_workspace_bytes(const sb_decoder_t* m) {
  if (!m) return 0;
  const size_t T = dl::kMaxT, H = m->hidden;
  const int G = 148 * 2;
  return T * H * 4 + 4 * T * H * 2 + T * (size_t)m->ffn * 2 + (H / 16) * T * 4 + (size_t)G * dl::kMaxB * 8 + 1024;
}

int sb_draft_loop(const sb_decoder_t* m, const sb_kvcache_t* kv, int32_t b, int32_t k, const int32_t* d1_ids,
                  const int32_t* d1_pos, const int32_t* slots, const int32_t* d_base, int32_t* v_ids, int32_t* ds_ids,
                  int32_t* ds_pos, void* workspace, size_t ws_bytes, void* sync_words, void* stream) {
  if (!m || !kv || b < 1 || k < 0 || !workspace || !sync_words) return SB_EINVAL;
  g_last_count = 0;
  if (!g_dl_enabled || k == 0) return SB_EUNSUPPORTED;
  const int H = m->hidden, hd = m->head_dim;
  if (m->arch != SB_ARCH_LLAMA || m->dtype != SB_BF16 || m->tp || hd != dl::kHd || m->n_heads * hd != H ||
      H % 64 || H > 1024 || m->ffn % H || m->vocab % 16 || 2 * b > dl::kMaxT || m->n_layers > dl::kMaxL ||
      m->n_heads % m->n_kv_heads)
    return SB_EUNSUPPORTED;
  const int CS = m->ffn / H;
  if (CS != 2 && CS != 4 && CS != 8) return SB_EUNSUPPORTED;
  const int G = draft_loop_grid(CS);
  if (G < CS) return SB_EUNSUPPORTED;
  if (sb_draft_loop_workspace_bytes(m) > ws_bytes) return SB_EWORKSPACE;
  int NS = 8;
  while (NS > 2 && dl_smem_bytes(H, NS) > kDlSmemMax) --NS;
  dl::Params p{};
  p.L = m->n_layers;
  p.H = H;
  p.nq = m->n_heads;
  p.nkv = m->n_kv_heads;
  p.ffn = m->ffn;
  p.V = m->vocab;
  p.max_pos = m->max_pos;
  p.ctx_max = kv->ctx_max;
  p.slots = kv->slots;
  p.b = b;
  p.k = k;
  p.G = G;
  p.CS = CS;
  p.NS = NS;
  p.eps = m->rms_eps;
  p.att_scale = 1.0f / sqrtf((float)hd);
  p.embed = (const __nv_bfloat16*)m->embed;
  p.lm_head = (const __nv_bfloat16*)m->lm_head;
  p.final_norm = (const __nv_bfloat16*)m->final_norm;
  for (int l = 0; l < m->n_layers; ++l) {
    p.attn_norm[l] = (const __nv_bfloat16*)m->attn_norm[l];
    p.mlp_norm[l] = (const __nv_bfloat16*)m->mlp_norm[l];
    p.w_qkv[l] = (const __nv_bfloat16*)m->w_qkv[l];
    p.w_o[l] = (const __nv_bfloat16*)m->w_o[l];
    p.w_gu[l] = (const __nv_bfloat16*)m->w_gu[l];
    p.w_down[l] = (const __nv_bfloat16*)m->w_down[l];
  }
  p.cosT = m->rope_cos;
  p.sinT = m->rope_sin;
  p.kc = (__nv_bfloat16*)kv->k;
  p.vc = (__nv_bfloat16*)kv->v;
  p.layer_kv = (size_t)kv->slots * m->n_kv_heads * kv->ctx_max * hd;
  p.d1_ids = d1_ids;
  p.d1_pos = d1_pos;
  p.slot = slots;
  p.d_base = d_base;
  p.v_ids = v_ids;
  p.ds_ids = ds_ids;
  p.ds_pos = ds_pos;
  char* w = (char*)workspace;
  const size_t T = dl::kMaxT;
  auto take = [&](size_t bytes) {
    char* r = w;
    w += (bytes + 255) / 256 * 256;
    return (void*)r;
  };
  p.resid = (float*)take(T * H * 4);
  p.xb = (__nv_bfloat16*)take(T * H * 2);
  p.qr = (__nv_bfloat16*)take(T * H * 2);
  p.attn = (__nv_bfloat16*)take(T * H * 2);
  p.act = (__nv_bfloat16*)take(T * (size_t)m->ffn * 2);
  p.npart = (float*)take((H / 16) * T * 4);
  p.am_val = (float*)take((size_t)G * dl::kMaxB * 4);
  p.am_idx = (int*)take((size_t)G * dl::kMaxB * 4);
  if ((size_t)(w - (char*)workspace) > ws_bytes) return SB_EWORKSPACE;
  p.bar_count = (unsigned long long*)sync_words;
  p.exit_count = (unsigned*)((char*)sync_words + 8);

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(dl::kThreads);
  cfg.dynamicSmemBytes = dl_smem_bytes(H, NS);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dl::draft_loop_kernel, p);
  if (e != cudaSuccess) return (int)e;
  g_last_count = 1;
  return 0;
}

}  // extern "C"
