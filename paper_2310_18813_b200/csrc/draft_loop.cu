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
constexpr int kMaxCS = 4;
constexpr int kMaxG = 160;   // grid (CTAs) upper bound: one per SM

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
  const uint8_t* wpk;   // packed weight tiles (sb_draft_loop_pack): per layer qkv | o | gate/up | down, then lm_head
  size_t tile_bytes, layer_bytes;
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
  __nv_bfloat16* xb;     // [kMaxT][H]   bf16(resid * next gain)
  __nv_bfloat16* qr;     // [kMaxT][H]   rotated q
  __nv_bfloat16* attn;   // [kMaxT][H]
  __nv_bfloat16* act;    // [kMaxT][ffn]
  float* npart;          // [H/16][kMaxT] sum of squares of the new residual per 16-column unit
  float* am_val;         // [G][kMaxB]
  int* am_idx;
  unsigned long long* bar_count;  // grid barrier (self-resetting)
  unsigned* exit_count;
  unsigned long long* trace;  // diagnostics (sb_debug_draft_trace): globaltimer per barrier, NULL = off
  int flags;  // experiments (SB_DL_FLAGS): bit 0 KV loads through L1, bit 1 q before KV, bit 2 L2 prefetch of the
              // step's weight tiles, bit 3 L2 prefetch of the KV history, bit 4 L2 prefetch of the winners' embeddings
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

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
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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
  // the residual unit (16 columns) this CTA owns, or -1: unit u = cid + r * NCL (round r < 2) belongs
  // to rank r of cluster cid -- it runs that unit's o_proj tile AND leads its down_proj reduction,
  // so the fp32 residual of the unit never leaves the CTA's shared memory
  __device__ int own_unit() const {
    const int u = cid + rank * NCL;
    return (rank < 2 && u < nE) ? u : -1;
  }
};

// qkv tile u -> weight row of its r-th row (RoPE pairs (d, d+32) in rows r, r+8)
__device__ __forceinline__ int qkv_row(int u, int r) {
  const int hs = u >> 2, j = u & 3;
  return hs * kHd + (r < 8 ? 8 * j + r : 32 + 8 * j + (r - 8));
}

// ------------------------------------------------------------------ packed weight tiles
// Every tile is 16 rows x H (bf16) stored contiguously, so ONE bulk copy moves it; inside a row the
// 16-byte chunk c sits at (c & ~7) | ((c ^ row) & 7) -- the 128B-swizzle pattern, which makes the
// consumers' ldmatrix phases (8 rows, one logical chunk) bank-conflict free without padding.
//   layer l: [qkv tiles nA][o tiles nC][gate/up tiles nD][down tiles nE x CS (unit-major, chunk-minor)]
//   then lm_head tiles nF
__device__ __forceinline__ uint32_t swz_chunk(int c, int row) { return (uint32_t)((c & ~7) | ((c ^ row) & 7)); }

__global__ void pack_kernel(const Params p, uint8_t* dst) {
  // one CTA per tile, 256 threads over its 16 x (H/8) chunks
  const int nA = (p.nq + 2 * p.nkv) * kHd / 16, nC = p.H / 16, nD = 2 * p.ffn / 16, nE = p.H / 16;
  const int per_layer = nA + nC + nD + nE * p.CS;
  int t = blockIdx.x;
  const __nv_bfloat16* W;
  size_t ld = p.H;
  int u, col0 = 0, kind;
  if (t < per_layer * p.L) {
    const int l = t / per_layer;
    u = t % per_layer;
    if (u < nA) {
      W = p.w_qkv[l];
      kind = 0;
    } else if ((u -= nA) < nC) {
      W = p.w_o[l];
      kind = 1;
    } else if ((u -= nC) < nD) {
      W = p.w_gu[l];
      kind = 1;
    } else {
      u -= nD;
      W = p.w_down[l];
      ld = p.ffn;
      col0 = (u % p.CS) * p.H;
      u /= p.CS;
      kind = 1;
    }
  } else {
    u = t - per_layer * p.L;
    W = p.lm_head;
    kind = 1;
  }
  const int cpr = p.H / 8;  // 16-byte chunks per row
  uint4* out = reinterpret_cast<uint4*>(dst + (size_t)blockIdx.x * p.tile_bytes);
  for (int e = threadIdx.x; e < 16 * cpr; e += blockDim.x) {
    const int r = e / cpr, c = e % cpr;
    const int row = kind == 0 ? qkv_row(u, r) : 16 * u + r;
    out[r * cpr + swz_chunk(c, r)] = *reinterpret_cast<const uint4*>(W + (size_t)row * ld + col0 + c * 8);
  }
}

// ------------------------------------------------------------------ producer
__device__ void producer(const Params& p, const Sched& S, uint8_t* ring, uint64_t* full, uint64_t* empty, int slot_bytes) {
  const uint64_t pol = l2_policy_evict_last();
  const uint32_t tb = (uint32_t)p.tile_bytes;
  int n = 0;
  auto put = [&](size_t tile) {
    const int s = n % p.NS;
    if (n >= p.NS) mbar_wait(&empty[s], ((n / p.NS) + 1) & 1);
    mbar_expect_tx(&full[s], tb);
    bulk_g2s(ring + (size_t)s * slot_bytes, p.wpk + tile * p.tile_bytes, tb, &full[s], pol);
    ++n;
  };
  const size_t nA = S.nA, nC = S.nC, nD = S.nD;
  const size_t per_layer = nA + nC + nD + (size_t)S.nE * p.CS;
  auto pf = [&](size_t tile) { prefetch_l2(p.wpk + tile * p.tile_bytes, tb); };
  for (int j = 0; j < p.k; ++j) {
    // the whole step's tiles of this CTA go to L2 first (HBM streams them while the latency-bound
    // phases run; the lm_head tiles are the bulk), then into the smem ring in consumption order
    for (int l = 0; l < p.L && (p.flags & 4); ++l) {
      const size_t base = (size_t)l * per_layer;
      for (int u = S.first(S.offA()); u < S.nA; u += S.G) pf(base + u);
      if (S.own_unit() >= 0) pf(base + nA + S.own_unit());
      for (int u = S.first(S.offD()); u < S.nD; u += S.G) pf(base + nA + nC + u);
      for (int u = S.cid; u < S.nE; u += S.NCL) pf(base + nA + nC + nD + (size_t)u * p.CS + S.rank);
    }
    if (p.flags & 4)
      for (int u = S.first(S.offF()); u < S.nF; u += S.G) pf((size_t)p.L * per_layer + u);
    for (int l = 0; l < p.L; ++l) {
      const size_t base = (size_t)l * per_layer;
      for (int u = S.first(S.offA()); u < S.nA; u += S.G) put(base + u);
      if (S.own_unit() >= 0) put(base + nA + S.own_unit());
      for (int u = S.first(S.offD()); u < S.nD; u += S.G) put(base + nA + nC + u);
      for (int u = S.cid; u < S.nE; u += S.NCL) put(base + nA + nC + nD + (size_t)u * p.CS + S.rank);
    }
    for (int u = S.first(S.offF()); u < S.nF; u += S.G) put((size_t)p.L * per_layer + u);
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
  float* rs;          // [kMaxT][16] fp32 residual of the owned unit
  float* cs;          // [kMaxT][kHd/2] RoPE cos of the step's positions
  float* sn;          // [kMaxT][kHd/2]
  int* slot;          // [kMaxB] KV slots
  __nv_bfloat16* g0;  // [H] attn_norm[0] (the embedding's consumer gain)
  float* gown;        // [kMaxL][2][16] owned unit's mlp_norm[l] / next-consumer gains
  float* amw;         // [8 warps][kMaxB] lm_head argmax partials (value)
  int* amwi;          // [8 warps][kMaxB] (index)
  uint64_t* full;
  uint64_t* empty;
  uint64_t* ebar;     // [2] cluster-reduce barriers (leader)
  int srow, xrow;
};

// diagnostics: CTA 0's timestamp of intra-phase point i (1: inputs staged, 2: tiles done) of the phase
// that ends at barrier nbar + 1
__device__ __forceinline__ void tmark(const Params& p, int nbar, int i) {
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && nbar < 511) p.trace[2048 + 4 * (nbar + 1) + i] = gtimer();
}

// grid barrier #idx (0-based over the launch): all G CTAs' consumer threads
__device__ __forceinline__ void grid_bar(const Params& p, int& nbar) {
  named_bar();
  ++nbar;
  if (threadIdx.x == 0) {
    // trace layout: [0] start, then per barrier i (1-based): [2i-1] CTA-0 arrival, [2i] CTA-0 exit;
    // per-CTA arrivals at [4096 + i * kMaxG + c]
    if (p.trace) {
      const unsigned long long t = gtimer();
      if (blockIdx.x == 0) p.trace[2 * nbar - 1] = t;
      if (nbar < 512) p.trace[4096 + (size_t)nbar * kMaxG + blockIdx.x] = t;
    }
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
    if (p.trace && blockIdx.x == 0) p.trace[2 * nbar] = gtimer();
  }
  named_bar();
}

// Stage a phase's inputs: X rows t < T of src (row t*row_step + row_off, stride ld) -> xs by
// cp.async (L2), and -- while those are in flight -- 1/rms per token from the producer partials
// npart[unit][row] (16 threads per token each sum every 16th unit, then a fixed-order half-warp
// tree: deterministic).  Ends with the consumer barrier.
__device__ __forceinline__ void stage(const Smem& sm, const Params& p, const __nv_bfloat16* src, int ld, int T,
                                      bool rinv, int nbar, int row_step = 1, int row_off = 0) {
  const int vec = p.H / 8;
  for (int e = threadIdx.x; e < T * vec; e += kConsumers) {
    const int t = e / vec, v = e % vec;
    cp_async16(sm.xs + (size_t)t * sm.xrow + v * 8, src + (size_t)(t * row_step + row_off) * ld + v * 8);
  }
  cp_async_commit();
  if (rinv) {
    const int nU = p.H / 16;
    const int t = threadIdx.x >> 4, j = threadIdx.x & 15;
    float ss = 0.f;
    if (t < T) {
      const float* src2 = p.npart + t * row_step + row_off;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (j + 16 * i < nU) v[i] = __ldcg(src2 + (j + 16 * i) * kMaxT);
      ss = (v[0] + v[1]) + (v[2] + v[3]);
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (t < T && j == 0) sm.rinv[t] = rsqrtf(ss / (float)p.H + p.eps);
  }
  cp_async_wait<0>();
  named_bar();
  tmark(p, nbar, 1);
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
  const int ar = lane & 15;
  const uint32_t wa = smem_u32(sm.ring + (size_t)s * 16 * sm.srow) + (uint32_t)(ar * sm.srow);
  const int tok = (lane & 7) + (lane >> 4) * 8;
  const uint32_t xa = smem_u32(sm.xs) + (uint32_t)((tok * sm.xrow + ((lane >> 3) & 1) * 8) * 2);
  const bool two = T > 8;
  for (int kk = k0; kk < k1; ++kk) {
    uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
    ldsm_x4(wa + swz_chunk(2 * kk + (lane >> 4), ar) * 16, a0, a1, a2, a3);
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

// Residual epilogue of the owned unit u (o_proj / down_proj): rs[t][r] += v (fp32, on chip);
// xb[t][16u + r] = bf16(new * gain); npart[u][t] = sum over the unit's 16 columns of new^2
__device__ __forceinline__ void resid_epilogue(const Params& p, const Smem& sm, float v, int u, int T,
                                               const float* gain16) {
  const int r = threadIdx.x & 15, t = threadIdx.x >> 4;
  float sq = 0.f;
  if (t < T) {
    const float nv = sm.rs[threadIdx.x] + v;
    sm.rs[threadIdx.x] = nv;
    p.xb[(size_t)t * p.H + 16 * u + r] = __float2bfloat16_rn(nv * gain16[r]);
    sq = nv * nv;
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (r == 0 && t < T) __stcg(p.npart + u * kMaxT + t, sq);
}

// Attention over the slot's cache for one (q head, sequence): q_len <= 2 queries, keys [0, pos].
// Warp w takes a contiguous key range in 32-key chunks.  Loads are coalesced 16-byte pieces: lane
// (g = lane / 8, c = lane % 8) holds dims 8c..8c+7 of key rows 4i + g (i < 8) for K and V alike, so a
// chunk is 8 + 8 load instructions per lane covering 32 full 128-byte rows each.  Scores reduce over
// the 8 lanes of a group; PV accumulates 8 dims per lane over its group's keys; groups merge at the end.
__device__ void attention_unit(const Params& p, const Smem& sm, int l, int h, int s, int q, const __nv_bfloat16* kc,
                               const __nv_bfloat16* vc, int nbar) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 3, c8 = lane & 7;
  const int t0 = s * q;
  const int hk = h / (p.nq / p.nkv);
  const int slot = sm.slot[s];
  const int pos_i[2] = {sm.tpos[t0], sm.tpos[t0 + q - 1]};
  const int n_keys = pos_i[1] + 1;
  const int per = (n_keys + 7) / 8;
  const int kb = warp * per, ke = min(n_keys, kb + per);
  const size_t slab = ((size_t)slot * p.nkv + hk) * p.ctx_max * kHd;
  const uint4* K = reinterpret_cast<const uint4*>(kc + slab) + c8;
  const uint4* Vv = reinterpret_cast<const uint4*>(vc + slab) + c8;
  uint4 kw[8], vw[8];
  auto load_chunk = [&](int base) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = base + 4 * i + g;
      const bool ok = row < ke;
      if (p.flags & 1) {
        kw[i] = ok ? K[(size_t)row * (kHd / 8)] : make_uint4(0, 0, 0, 0);
        vw[i] = ok ? Vv[(size_t)row * (kHd / 8)] : make_uint4(0, 0, 0, 0);
      } else {
        kw[i] = ok ? __ldcg(K + (size_t)row * (kHd / 8)) : make_uint4(0, 0, 0, 0);
        vw[i] = ok ? __ldcg(Vv + (size_t)row * (kHd / 8)) : make_uint4(0, 0, 0, 0);
      }
    }
  };
  if (kb < ke && !(p.flags & 2)) load_chunk(kb);  // in flight while the queries are staged
  for (int e = threadIdx.x; e < q * kHd; e += kConsumers) {
    const int i = e / kHd, d = e % kHd;
    sm.qs[i * kHd + d] = __bfloat162float(__ushort_as_bfloat16(
        __ldcg(reinterpret_cast<const unsigned short*>(p.qr) + (size_t)(t0 + i) * p.H + h * kHd + d)));
  }
  named_bar();
  if (kb < ke && (p.flags & 2)) load_chunk(kb);
  tmark(p, nbar, 1);
  float qv[2][8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    qv[0][e] = sm.qs[8 * c8 + e];
    qv[1][e] = q > 1 ? sm.qs[kHd + 8 * c8 + e] : 0.f;
  }
  float m[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f};
  float o[2][8];
#pragma unroll
  for (int e = 0; e < 8; ++e) o[0][e] = o[1][e] = 0.f;
  for (int base = kb; base < ke; base += 32) {
    if (base != kb) load_chunk(base);
    float sc[2][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&kw[i]);
      float d0 = 0.f, d1 = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(hv[e]);
        d0 += f.x * qv[0][2 * e] + f.y * qv[0][2 * e + 1];
        d1 += f.x * qv[1][2 * e] + f.y * qv[1][2 * e + 1];
      }
#pragma unroll
      for (int o_ = 1; o_ < 8; o_ <<= 1) {
        d0 += __shfl_xor_sync(0xffffffffu, d0, o_);
        d1 += __shfl_xor_sync(0xffffffffu, d1, o_);
      }
      const int row = base + 4 * i + g;
      sc[0][i] = (row < ke && row <= pos_i[0]) ? d0 * p.att_scale : -INFINITY;
      sc[1][i] = (q > 1 && row < ke && row <= pos_i[1]) ? d1 * p.att_scale : -INFINITY;
    }
#pragma unroll
    for (int qi = 0; qi < 2; ++qi) {
      float cm = sc[qi][0];
#pragma unroll
      for (int i = 1; i < 8; ++i) cm = fmaxf(cm, sc[qi][i]);
      cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 8));
      cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 16));
      const float nm = fmaxf(m[qi], cm);
      const float corr = nm == -INFINITY ? 1.f : __expf(m[qi] - nm);
      float ls = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) o[qi][e] *= corr;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float pr = sc[qi][i] == -INFINITY ? 0.f : __expf(sc[qi][i] - nm);
        ls += pr;
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&vw[i]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(hv[e]);
          o[qi][2 * e] += pr * f.x;
          o[qi][2 * e + 1] += pr * f.y;
        }
      }
      ls += __shfl_xor_sync(0xffffffffu, ls, 8);
      ls += __shfl_xor_sync(0xffffffffu, ls, 16);
      lsum[qi] = lsum[qi] * corr + ls;
      m[qi] = nm;
    }
  }
  // merge the 4 lane groups (each holds its keys' PV for dims 8c..8c+7)
#pragma unroll
  for (int qi = 0; qi < 2; ++qi)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      o[qi][e] += __shfl_xor_sync(0xffffffffu, o[qi][e], 8);
      o[qi][e] += __shfl_xor_sync(0xffffffffu, o[qi][e], 16);
    }
  tmark(p, nbar, 3);
  float* aw = sm.att + (size_t)warp * 2 * (kHd + 2);
  if (g == 0) {
#pragma unroll
    for (int qi = 0; qi < 2; ++qi) {
#pragma unroll
      for (int e = 0; e < 8; ++e) aw[qi * (kHd + 2) + 8 * c8 + e] = o[qi][e];
      if (c8 == 0) {
        aw[qi * (kHd + 2) + kHd] = m[qi];
        aw[qi * (kHd + 2) + kHd + 1] = lsum[qi];
      }
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
__device__ void embed_step(const Params& p, const Smem& sm, int own, int T) {
  // every load of the step in flight at once: raw embedding rows -> xs, RoPE cos/sin rows of the
  // step's positions -> smem (the qkv epilogue's), by cp.async
  const int vec = p.H / 8;
  for (int e = threadIdx.x; e < T * vec; e += kConsumers) {
    const int t = e / vec, v = e % vec;
    const int id = sm.tid_tok[t];
    const bool pad = sm.tpos[t] < 0 || id < 0 || id >= p.V;
    cp_async16(sm.xs + (size_t)t * sm.xrow + v * 8, p.embed + (size_t)(pad ? 0 : id) * p.H + v * 8);
  }
  for (int e = threadIdx.x; e < 2 * T * (kHd / 8); e += kConsumers) {  // 8 x 16 B per (table, token)
    const int tab = e / (T * (kHd / 8)), r = e % (T * (kHd / 8)), t = r / (kHd / 8), v = r % (kHd / 8);
    const int pos = sm.tpos[t];
    const int pc = pos < 0 ? 0 : (pos >= p.max_pos ? p.max_pos - 1 : pos);
    cp_async16((tab ? sm.sn : sm.cs) + t * (kHd / 2) + v * 4, (tab ? p.sinT : p.cosT) + (size_t)pc * (kHd / 2) + v * 4);
  }
  cp_async_commit();
  cp_async_wait<0>();
  named_bar();
  // the fp32 residual of the owned unit starts as the embedding (kept on chip for the whole step)
  if (own >= 0 && (int)threadIdx.x < T * 16) {
    const int t = threadIdx.x >> 4, col = 16 * own + (threadIdx.x & 15);
    const bool pad = sm.tpos[t] < 0 || sm.tid_tok[t] < 0 || sm.tid_tok[t] >= p.V;
    sm.rs[threadIdx.x] = pad ? 0.f : __bfloat162float(sm.xs[(size_t)t * sm.xrow + col]);
  }
  named_bar();
  // 16 threads per token: sum of squares of its 16-byte chunks j, j+16, ... (fixed-order half-warp
  // tree), then the same chunks scaled in place by the attn_norm[0] gain -> the qkv GEMM input
  const int t = threadIdx.x >> 4, j = threadIdx.x & 15;
  const __nv_bfloat16* g = sm.g0;
  float ss = 0.f;
  const bool pad = t < T && (sm.tpos[t] < 0 || sm.tid_tok[t] < 0 || sm.tid_tok[t] >= p.V);
  if (t < T) {
    for (int v = j; v < vec; v += 16) {
      uint4 w = *reinterpret_cast<const uint4*>(sm.xs + (size_t)t * sm.xrow + v * 8);
      if (pad) w = make_uint4(0, 0, 0, 0);
      const uint4 gw = *reinterpret_cast<const uint4*>(g + v * 8);
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
      *reinterpret_cast<uint4*>(sm.xs + (size_t)t * sm.xrow + v * 8) = outw;
    }
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (t < T && j == 0) sm.rinv[t] = rsqrtf(ss / (float)p.H + p.eps);
  named_bar();
}

__global__ void __launch_bounds__(kThreads, 1) draft_loop_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int H = p.H;
  Smem sm;
  sm.srow = H * 2;
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
  sm.qs = sm.red;                   // (attention never overlaps a tile reduction: alias)
  sm.att = sm.red + 2 * kHd;
  sm.cs = reinterpret_cast<float*>(q);
  q += kMaxT * (kHd / 2) * 4;
  sm.sn = reinterpret_cast<float*>(q);
  q += kMaxT * (kHd / 2) * 4;
  sm.slot = reinterpret_cast<int*>(q);
  q += kMaxB * 4;
  sm.g0 = reinterpret_cast<__nv_bfloat16*>(q);
  q += (size_t)H * 2;
  sm.gown = reinterpret_cast<float*>(q);
  q += kMaxL * 2 * 16 * 4;
  sm.rinv = reinterpret_cast<float*>(q);
  q += kMaxT * 4;
  sm.tid_tok = reinterpret_cast<int*>(q);
  q += kMaxT * 4;
  sm.tpos = reinterpret_cast<int*>(q);
  q += kMaxT * 4;
  sm.tok_next = reinterpret_cast<int*>(q);
  q += kMaxB * 4;
  sm.rs = reinterpret_cast<float*>(q);
  q += kMaxT * 16 * 4;
  sm.amw = reinterpret_cast<float*>(q);
  q += 8 * kMaxB * 4;
  sm.amwi = reinterpret_cast<int*>(q);
  q += 8 * kMaxB * 4;
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
    if (threadIdx.x == kConsumers) producer(p, S, sm.ring, sm.full, sm.empty, 16 * sm.srow);  // weights: no dependency
    return;
  }
  griddep_wait();  // committed tokens / staging written by the previous kernels
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[0] = gtimer();
  if ((int)threadIdx.x < p.b) sm.slot[threadIdx.x] = p.slot[threadIdx.x];
  for (int i = threadIdx.x; i < H; i += kConsumers) sm.g0[i] = p.attn_norm[0][i];
  if (S.own_unit() >= 0)
    for (int i = threadIdx.x; i < p.L * 32; i += kConsumers) {
      const int l = i >> 5, which = (i >> 4) & 1, r = i & 15;
      const __nv_bfloat16* gsrc = which == 0 ? p.mlp_norm[l] : (l + 1 < p.L ? p.attn_norm[l + 1] : p.final_norm);
      sm.gown[i] = __bfloat162float(gsrc[16 * S.own_unit() + r]);
    }
  const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = p.b;
  int n = 0, nbar = 0;
  int e_use[2] = {0, 0};
  const int own = S.own_unit();
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
    if (tid == 0 && (p.flags & 8)) {  // the KV history this CTA's attention units will read, every layer, into L2
      for (int un = c; un < p.nq * b; un += S.G) {
        const int s_ = un / p.nq, hk = (un % p.nq) / (p.nq / p.nkv);
        const int nk = sm.tpos[s_ * qn + qn - 1] + 1;
        const size_t off = ((size_t)sm.slot[s_] * p.nkv + hk) * p.ctx_max * kHd;
        for (int l = 0; l < p.L; ++l) {
          prefetch_l2(p.kc + (size_t)l * p.layer_kv + off, (uint32_t)nk * kHd * 2);
          prefetch_l2(p.vc + (size_t)l * p.layer_kv + off, (uint32_t)nk * kHd * 2);
        }
      }
    }
    named_bar();
    embed_step(p, sm, own, T);
    tmark(p, nbar, 1);
    for (int l = 0; l < p.L; ++l) {
      const __nv_bfloat16* kcl = p.kc + (size_t)l * p.layer_kv;
      const __nv_bfloat16* vcl = p.vc + (size_t)l * p.layer_kv;
      // ---- A: qkv + 1/rms + RoPE + KV append
      if (l > 0 && S.first(S.offA()) < S.nA) stage(sm, p, p.xb, H, T, true, nbar);
      for (int u = S.first(S.offA()); u < S.nA; u += S.G) {
        const float acc = tile_mma(sm, H, p.NS, n, T);
        const int r = tid & 15, t = tid >> 4;
        const float v = t < T ? __bfloat162float(__float2bfloat16_rn(acc * sm.rinv[t])) : 0.f;
        const float partner = __shfl_xor_sync(0xffffffffu, v, 8);
        const int hs = u >> 2, jj = u & 3;
        const int i = 8 * jj + (r & 7);  // rotary pair index (dims i, i + 32)
        if (t < T) {
          const int pos = sm.tpos[t];
          const int d = qkv_row(u, r) - hs * kHd;
          float out = v;
          if (hs < p.nq + p.nkv) {  // q or k: rotate-half
            const float cs = sm.cs[t * (kHd / 2) + i], sn = sm.sn[t * (kHd / 2) + i];
            out = r < 8 ? v * cs - partner * sn : v * cs + partner * sn;
          }
          const __nv_bfloat16 ob = __float2bfloat16_rn(out);
          if (hs < p.nq) {
            p.qr[(size_t)t * H + hs * kHd + d] = ob;
          } else if (pos >= 0) {
            const int s = t / qn;
            const int kvh = hs < p.nq + p.nkv ? hs - p.nq : hs - p.nq - p.nkv;
            __nv_bfloat16* dst = (hs < p.nq + p.nkv ? p.kc : p.vc) + (size_t)l * p.layer_kv +
                                 (((size_t)sm.slot[s] * p.nkv + kvh) * p.ctx_max + pos) * kHd + d;
            *dst = ob;
          }
        }
      }
      tmark(p, nbar, 2);
      tmark(p, nbar, 2);
    grid_bar(p, nbar);
      // ---- B: attention (causal inside the window)
      for (int un = c; un < p.nq * b; un += S.G) attention_unit(p, sm, l, un % p.nq, un / p.nq, qn, kcl, vcl, nbar);
      tmark(p, nbar, 2);
      tmark(p, nbar, 2);
    grid_bar(p, nbar);
      // ---- C: o_proj of the owned unit (+ residual on chip, bf16 copy * mlp gain, norm partials)
      if (own >= 0) {
        stage(sm, p, p.attn, H, T, false, nbar);
        const float acc = tile_mma(sm, H, p.NS, n, T);
        resid_epilogue(p, sm, acc, own, T, sm.gown + l * 32);
      }
      tmark(p, nbar, 2);
      tmark(p, nbar, 2);
    grid_bar(p, nbar);
      // ---- D: gate/up (interleaved rows) -> silu(g) * u
      if (S.first(S.offD()) < S.nD) stage(sm, p, p.xb, H, T, true, nbar);
      for (int u = S.first(S.offD()); u < S.nD; u += S.G) {
        const float acc = tile_mma(sm, H, p.NS, n, T);
        const int r = tid & 15, t = tid >> 4;
        const float v = t < T ? acc * sm.rinv[t] : 0.f;
        const float up = __shfl_xor_sync(0xffffffffu, v, 1);
        if (t < T && !(r & 1)) p.act[(size_t)t * p.ffn + 8 * u + (r >> 1)] = __float2bfloat16_rn(silu(v) * up);
      }
      tmark(p, nbar, 2);
      tmark(p, nbar, 2);
    grid_bar(p, nbar);
      // ---- E: down_proj, K split over the cluster ranks; unit u = cid + r*NCL is reduced in rank
      // order at its owner (rank r), which also holds its residual
      if (S.cid < S.nE) stage(sm, p, p.act + (size_t)S.rank * H, p.ffn, T, false, nbar);
      {
        for (int rd = 0, u = S.cid; u < S.nE; u += S.NCL, ++rd) {
          const float acc = tile_mma(sm, H, p.NS, n, T);
          float* dp = sm.dpart + (size_t)rd * kMaxCS * kMaxT * 16;
          if (S.rank == rd) {
            dp[S.rank * kMaxT * 16 + tid] = acc;
            mbar_wait_cluster(&sm.ebar[rd], e_use[rd] & 1);
            ++e_use[rd];
            float v = 0.f;
            for (int r = 0; r < p.CS; ++r) v += dp[r * kMaxT * 16 + tid];
            resid_epilogue(p, sm, v, u, T, sm.gown + l * 32 + 16);
          } else {
            st_cluster_f32(map_rank(smem_u32(dp + S.rank * kMaxT * 16 + tid), rd), acc);
            named_bar();
            if (tid == 0) mbar_arrive_remote(map_rank(smem_u32(&sm.ebar[rd]), rd));
          }
        }
      }
      tmark(p, nbar, 2);
      tmark(p, nbar, 2);
    grid_bar(p, nbar);
    }
    // ---- F: lm_head over the last token of each sequence, fused 1/rms + argmax; one tile per warp
    // (warp w takes this CTA's tiles w, w + NS, ... -- always ring slot (n0 + w) % NS), no cross-warp
    // reduction per tile; warps merge their running (max, index) once at the end
    if (S.first(S.offF()) < S.nF) stage(sm, p, p.xb, H, b, true, nbar, qn, qn - 1);
    {
      const int n0 = n;
      const int f0 = S.first(S.offF());
      const int cnt = f0 < S.nF ? (S.nF - 1 - f0) / S.G + 1 : 0;
      ArgMax r0{-INFINITY, INT_MAX}, r1{-INFINITY, INT_MAX};
      const int g = lane >> 2, q2 = (lane & 3) * 2;
      const float ri0 = q2 < b ? sm.rinv[q2] : 0.f, ri1 = q2 + 1 < b ? sm.rinv[q2 + 1] : 0.f;
      if (warp < p.NS) {
        const uint32_t xa = smem_u32(sm.xs) + (uint32_t)((((lane & 7) + (lane >> 4) * 8) * sm.xrow + ((lane >> 3) & 1) * 8) * 2);
        for (int li = warp; li < cnt; li += p.NS) {
          const int u = f0 + li * S.G;
          const int nn = n0 + li, sl = nn % p.NS;
          mbar_wait(&sm.full[sl], (nn / p.NS) & 1);
          const int ar = lane & 15;
          const uint32_t wa = smem_u32(sm.ring + (size_t)sl * 16 * sm.srow) + (uint32_t)(ar * sm.srow);
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
          for (int kk = 0; kk < H / 16; ++kk) {
            uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
            ldsm_x4(wa + swz_chunk(2 * kk + (lane >> 4), ar) * 16, a0, a1, a2, a3);
            ldsm_x4(xa + kk * 32, b0, b1, b2, b3);
            mma_bf16(acc, a0, a1, a2, a3, b0, b1);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.empty[sl]);
          ArgMax x0 = argmax_merge(ArgMax{q2 < b ? acc[0] * ri0 : -INFINITY, 16 * u + g},
                                   ArgMax{q2 < b ? acc[2] * ri0 : -INFINITY, 16 * u + g + 8});
          ArgMax x1 = argmax_merge(ArgMax{q2 + 1 < b ? acc[1] * ri1 : -INFINITY, 16 * u + g},
                                   ArgMax{q2 + 1 < b ? acc[3] * ri1 : -INFINITY, 16 * u + g + 8});
#pragma unroll
          for (int o = 4; o < 32; o <<= 1) {
            x0 = argmax_merge(x0, ArgMax{__shfl_xor_sync(0xffffffffu, x0.v, o), __shfl_xor_sync(0xffffffffu, x0.i, o)});
            x1 = argmax_merge(x1, ArgMax{__shfl_xor_sync(0xffffffffu, x1.v, o), __shfl_xor_sync(0xffffffffu, x1.i, o)});
          }
          r0 = argmax_merge(r0, x0);
          r1 = argmax_merge(r1, x1);
        }
      }
      n = n0 + cnt;
      if (lane < 4) {
        sm.amw[warp * kMaxB + q2] = r0.v;
        sm.amwi[warp * kMaxB + q2] = r0.i;
        sm.amw[warp * kMaxB + q2 + 1] = r1.v;
        sm.amwi[warp * kMaxB + q2 + 1] = r1.i;
      }
      named_bar();
      if (tid < b) {
        ArgMax a{-INFINITY, INT_MAX};
        for (int w = 0; w < 8; ++w) a = argmax_merge(a, ArgMax{sm.amw[w * kMaxB + tid], sm.amwi[w * kMaxB + tid]});
        __stcg(p.am_val + c * kMaxB + tid, a.v);
        __stcg(p.am_idx + c * kMaxB + tid, a.i);
        // the global winner is one of the CTAs' local winners: its embedding row (the next step's
        // input) heads for L2 now, not after the argmax
        if ((p.flags & 16) && j < p.k && a.i >= 0 && a.i < p.V) prefetch_l2(p.embed + (size_t)a.i * p.H, (uint32_t)p.H * 2);
      }
    }
    tmark(p, nbar, 2);
    grid_bar(p, nbar);
    // ---- G: argmax over the CTA partials -> d_j (every CTA: the next step's tokens)
    if (warp < b) {
      ArgMax a{-INFINITY, INT_MAX};
      float vv[kMaxG / 32];
      int ii[kMaxG / 32];
#pragma unroll
      for (int i = 0; i < kMaxG / 32; ++i) {
        const int cc = lane + 32 * i;
        vv[i] = cc < S.G ? __ldcg(p.am_val + cc * kMaxB + warp) : -INFINITY;
        ii[i] = cc < S.G ? __ldcg(p.am_idx + cc * kMaxB + warp) : INT_MAX;
      }
#pragma unroll
      for (int i = 0; i < kMaxG / 32; ++i)
        if (vv[i] != -INFINITY) a = argmax_merge(a, ArgMax{vv[i], ii[i]});  // (-inf: a CTA without lm_head tiles)
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

// Off by default: with the templated per-step kernels (small, instruction-cache resident) the per-step
// forwards are faster at every b <= 8, k (profiles/r2/draft_loop_vs_per_step_r2c.txt: b=8,k=3 186 vs
// 196 us, b=1,k=8 442 vs 446 us); sb_set_draft_loop(1) opts in.
static int g_dl_enabled = 0;
static unsigned long long* g_dl_trace = nullptr;
static int g_dl_clusters[9] = {0};  // max co-resident clusters per cluster size (1 CTA per SM)

static size_t dl_smem_bytes(int H, int NS) {
  size_t b = (size_t)NS * 16 * (H * 2) + (size_t)dl::kMaxT * (H + 8) * 2 + 2 * 8 * dl::kMaxT * 16 * 4 +
             2 * dl::kMaxCS * dl::kMaxT * 16 * 4 + 3 * dl::kMaxT * 4 + dl::kMaxB * 4 + 16;
  b += dl::kMaxT * 16 * 4 + 2 * 8 * dl::kMaxB * 4;           // rs, amw, amwi
  b += 2 * dl::kMaxT * (dl::kHd / 2) * 4 + dl::kMaxB * 4;    // cos / sin rows, slots
  b += (size_t)H * 2 + dl::kMaxL * 2 * 16 * 4;                // gains
  return b + (size_t)(2 * NS + 2) * 8;
}
constexpr size_t kDlSmemMax = 227 * 1024;

// L2 residency of the draft's weights: its evict-last stream (the packed tiles, re-read every draft
// step) only sticks inside the persisting carve-out, which is 0 unless the process sets it.
static size_t g_dl_persist = 0;

int draft_loop_init() {
  {
    const char* env = getenv("SB_DL_PERSIST_MB");
    const long want_mb = env ? atol(env) : 0;  // measured: no gain for the draft, and it shrinks the target's L2
    int dev = 0, max_persist = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    size_t want = (size_t)want_mb << 20;
    if (want > (size_t)max_persist) want = (size_t)max_persist;
    if (want > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) g_dl_persist = want;
    cudaGetLastError();
  }
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

int sb_debug_draft_trace(void* buf) {
  g_dl_trace = (unsigned long long*)buf;
  return 0;
}

int sb_set_draft_loop(int32_t enabled) {
  g_dl_enabled = enabled ? 1 : 0;
  return 0;
}

size_t sb_draft_loop_workspace_bytes(const sb_decoder_t* m) {
  if (!m) return 0;
  const size_t T = dl::kMaxT, H = m->hidden;
  return T * H * 4 + 4 * T * H * 2 + T * (size_t)m->ffn * 2 + (H / 16) * T * 4 + (size_t)dl::kMaxG * dl::kMaxB * 8 +
         4096;
}

// The envelope of the kernel and the weight part of its parameters (shared by pack and launch).
static int dl_setup(const sb_decoder_t* m, dl::Params* p) {
  const int H = m->hidden, hd = m->head_dim;
  if (m->arch != SB_ARCH_LLAMA || m->dtype != SB_BF16 || m->tp || hd != dl::kHd || m->n_heads * hd != H ||
      H % 64 || H > 1024 || m->ffn % H || m->vocab % 16 || m->n_layers > dl::kMaxL || m->n_heads % m->n_kv_heads)
    return SB_EUNSUPPORTED;
  const int CS = m->ffn / H;
  if (CS != 2 && CS != 4) return SB_EUNSUPPORTED;
  int G = draft_loop_grid(CS);
  if (G > dl::kMaxG) G = dl::kMaxG / CS * CS;
  if (G < CS) return SB_EUNSUPPORTED;
  if ((H / 16 + G / CS - 1) / (G / CS) > 2) return SB_EUNSUPPORTED;  // <= 2 down_proj rounds (owned units)
  *p = dl::Params{};
  p->L = m->n_layers;
  p->H = H;
  p->nq = m->n_heads;
  p->nkv = m->n_kv_heads;
  p->ffn = m->ffn;
  p->V = m->vocab;
  p->max_pos = m->max_pos;
  p->G = G;
  p->CS = CS;
  p->eps = m->rms_eps;
  p->att_scale = 1.0f / sqrtf((float)hd);
  p->embed = (const __nv_bfloat16*)m->embed;
  p->lm_head = (const __nv_bfloat16*)m->lm_head;
  p->final_norm = (const __nv_bfloat16*)m->final_norm;
  for (int l = 0; l < m->n_layers; ++l) {
    p->attn_norm[l] = (const __nv_bfloat16*)m->attn_norm[l];
    p->mlp_norm[l] = (const __nv_bfloat16*)m->mlp_norm[l];
    p->w_qkv[l] = (const __nv_bfloat16*)m->w_qkv[l];
    p->w_o[l] = (const __nv_bfloat16*)m->w_o[l];
    p->w_gu[l] = (const __nv_bfloat16*)m->w_gu[l];
    p->w_down[l] = (const __nv_bfloat16*)m->w_down[l];
  }
  p->cosT = m->rope_cos;
  p->sinT = m->rope_sin;
  p->tile_bytes = (size_t)16 * H * 2;
  const size_t nA = (size_t)(m->n_heads + 2 * m->n_kv_heads) * hd / 16;
  p->layer_bytes = (nA + H / 16 + 2 * (size_t)m->ffn / 16 + (size_t)(H / 16) * CS) * p->tile_bytes;
  return 0;
}

size_t sb_draft_loop_packed_bytes(const sb_decoder_t* m) {
  dl::Params p;
  if (!m || dl_setup(m, &p)) return 0;
  return p.layer_bytes * p.L + (size_t)(p.V / 16) * p.tile_bytes;
}

int sb_draft_loop_pack(const sb_decoder_t* m, void* dst, size_t bytes, void* stream) {
  if (!m || !dst) return SB_EINVAL;
  dl::Params p;
  SB_TRY(dl_setup(m, &p));
  const size_t need = p.layer_bytes * p.L + (size_t)(p.V / 16) * p.tile_bytes;
  if (bytes < need) return SB_EWORKSPACE;
  const int tiles = (int)(need / p.tile_bytes);
  dl::pack_kernel<<<tiles, 256, 0, (cudaStream_t)stream>>>(p, (uint8_t*)dst);
  SB_CHECK_LAUNCH();
  return 0;
}

int sb_draft_loop(const sb_decoder_t* m, const sb_kvcache_t* kv, const void* packed, int32_t b, int32_t k,
                  const int32_t* d1_ids, const int32_t* d1_pos, const int32_t* slots, const int32_t* d_base,
                  int32_t* v_ids, int32_t* ds_ids, int32_t* ds_pos, void* workspace, size_t ws_bytes,
                  void* sync_words, void* stream) {
  if (!m || !kv || b < 1 || k < 0 || !workspace || !sync_words) return SB_EINVAL;
  g_last_count = 0;
  if (!g_dl_enabled || k == 0 || 2 * b > dl::kMaxT) return SB_EUNSUPPORTED;
  dl::Params p;
  SB_TRY(dl_setup(m, &p));
  if (!packed) return SB_EINVAL;
  if (sb_draft_loop_workspace_bytes(m) > ws_bytes) return SB_EWORKSPACE;
  const int H = p.H;
  int NS = 8;
  while (NS > 2 && dl_smem_bytes(H, NS) > kDlSmemMax) --NS;
  p.NS = NS;
  p.ctx_max = kv->ctx_max;
  p.slots = kv->slots;
  p.b = b;
  p.k = k;
  p.wpk = (const uint8_t*)packed;
  p.kc = (__nv_bfloat16*)kv->k;
  p.vc = (__nv_bfloat16*)kv->v;
  p.layer_kv = (size_t)kv->slots * m->n_kv_heads * kv->ctx_max * dl::kHd;
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
  p.xb = (__nv_bfloat16*)take(T * H * 2);
  p.qr = (__nv_bfloat16*)take(T * H * 2);
  p.attn = (__nv_bfloat16*)take(T * H * 2);
  p.act = (__nv_bfloat16*)take(T * (size_t)m->ffn * 2);
  p.npart = (float*)take((H / 16) * T * 4);
  p.am_val = (float*)take((size_t)dl::kMaxG * dl::kMaxB * 4);
  p.am_idx = (int*)take((size_t)dl::kMaxG * dl::kMaxB * 4);
  if ((size_t)(w - (char*)workspace) > ws_bytes) return SB_EWORKSPACE;
  p.bar_count = (unsigned long long*)sync_words;
  p.exit_count = (unsigned*)((char*)sync_words + 8);
  p.trace = g_dl_trace;
  {
    static int flags = -1;
    if (flags < 0) flags = getenv("SB_DL_FLAGS") ? atoi(getenv("SB_DL_FLAGS")) : 0;
    p.flags = flags;
  }

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(dl::kThreads);
  cfg.dynamicSmemBytes = dl_smem_bytes(H, NS);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.CS;
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
