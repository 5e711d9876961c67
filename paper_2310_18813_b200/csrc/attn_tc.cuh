// Tensor-core flash-decoding attention item (K3): the body of
// attention_tc_kernel (layer_kernels.cu) for speculative windows (RoPE + KV
// append fused) and, in block mode, for prefill-sized windows.
#pragma once
#include <climits>

#include "common.cuh"
#include "mma_ptx.cuh"

namespace sb {

constexpr int kTcKT = 64;

__device__ __forceinline__ void attn_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <int HD, int STAGES = 3>
struct TcAttnSmem {
  static constexpr int RS = HD + 8;                             // padded row (elements)
  static constexpr size_t tile = (size_t)kTcKT * RS * 2;        // one K or V tile
  static constexpr size_t stage = 2 * tile;
  static constexpr size_t q = (size_t)16 * RS * 2;
  static constexpr size_t comb = (size_t)4 * 16 * HD * 4 + 4 * 16 * 2 * 4;  // warp partials (aliases the ring)
  static constexpr size_t ring = STAGES * stage;
  static constexpr size_t bytes = q + (ring > comb ? ring : comb);
};

// Flash-decoding key splits (gridDim.z = n_splits > 1): split z takes an even
// share of the 64-key tiles, appends only the window rows inside its own key
// range (no cross-split dependency), and publishes an unnormalised partial
// (O, running max M, sum L per query row); the last split to finish (per-(seq,
// kv head) counter) merges the partials in split order -- deterministic -- and
// resets the counter for the next launch / graph replay.
struct AttnSplit {
  float* part;   // [n_seq][nkv][S][16][HD]
  float* ml;     // [n_seq][nkv][S][16][2]
  int* counter;  // [n_seq][nkv], zero between launches
};

struct AttnArgs {
  const __nv_bfloat16* qkv;
  __nv_bfloat16* kc;  // this layer's K cache base
  __nv_bfloat16* vc;
  __nv_bfloat16* out;
  const int32_t* tok_slot;
  const int32_t* tok_pos;
  const float* cosT;
  const float* sinT;
  int q_len, nq, nkv, ctx_max, max_pos;
  float scale;
  AttnSplit sp;
  const char* l2_next;  // next GEMM's weights: prefetched into L2 while this latency-bound kernel runs
  unsigned long long l2_next_bytes;
  // prefill blocks: Q already rotated by rope_append (qr [T][nq][HD]) and the
  // window already in the cache; CTA z takes tokens [z*q_blk, (z+1)*q_blk)
  const __nv_bfloat16* qr;
  int q_blk;
  int kv_evict_first;  // KV history streamed with an L2 evict-first policy (the target's cache)
  unsigned long long* trace;  // sb_debug_cta_trace (NULL = off)
  int trace_id;
  unsigned long long* tr_t;   // this CTA's stamps (shared memory)
};
struct AttnShared {
  int qpos[16], qtok[16], qhead[16];
  int wpos[16];  // this forward's positions for the sequence (the window keys)
  int last;
};

// One (kv head, sequence[, key split]) item on 128 threads (tid 0..127, named
// barrier 1): the body of attention_tc_kernel.  `pdl`: issue the
// KV-history tiles, then griddepcontrol.wait / launch_dependents.
template <int HD, int STAGES, bool BLK, bool SPLIT>
__device__ __forceinline__ void attn_tc_item(const AttnArgs& A, int kvh, int seq, int split, int n_splits,
                                             uint8_t* tsm, AttnShared& sh, int tid, bool pdl, int qb = 0) {
  const __nv_bfloat16* __restrict__ qkv = A.qkv;
  __nv_bfloat16* __restrict__ kc = A.kc;
  __nv_bfloat16* __restrict__ vc = A.vc;
  __nv_bfloat16* __restrict__ out = A.out;
  const int32_t* __restrict__ tok_slot = A.tok_slot;
  const int32_t* __restrict__ tok_pos = A.tok_pos;
  const float* __restrict__ cosT = A.cosT;
  const float* __restrict__ sinT = A.sinT;
  const int q_len = A.q_len, nq = A.nq, nkv = A.nkv, ctx_max = A.ctx_max, max_pos = A.max_pos;
  const float scale = A.scale;
  const AttnSplit& sp = A.sp;
  using SM = TcAttnSmem<HD, STAGES>;
  constexpr int RS = SM::RS, HALF = HD / 2, KSTEP = HD / 16, NT = HD / 8;
  constexpr int kTcStages = STAGES;
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(tsm);
  uint8_t* ring = tsm + SM::q;
  int* qpos = sh.qpos;
  int* qtok = sh.qtok;
  int* qhead = sh.qhead;

  const int group = nq / nkv;
  constexpr bool blk = BLK;  // prefill block of an already rotated / appended window (A.qr)
  const int t0 = blk ? qb * A.q_blk : 0;
  const int nQ = group * (blk ? min(A.q_blk, q_len - t0) : q_len);
  const int warp = tid >> 5, lane = tid & 31;
  // Before the programmatic-dependency wait only data written >= 2 kernels
  // back is touched (positions, slots, KV history): every kernel of the
  // engine triggers its dependents after its own wait, so the kernel two
  // launches back has completed.
  const int slot = tok_slot[seq];
  const int row_w = (nq + 2 * nkv) * HD;
  const __nv_bfloat16* seq_rows = qkv + (size_t)seq * q_len * row_w;
  __nv_bfloat16* kslab = kc + ((size_t)slot * nkv + kvh) * ctx_max * HD;
  __nv_bfloat16* vslab = vc + ((size_t)slot * nkv + kvh) * ctx_max * HD;

  if (tid < 16) {
    int t = tid / group;
    qtok[tid] = tid < nQ ? t0 + t : 0;
    qhead[tid] = kvh * group + tid % group;
    qpos[tid] = tid < nQ ? tok_pos[seq * q_len + t0 + t] : -1;
    sh.wpos[tid] = !blk && tid < q_len ? tok_pos[seq * q_len + tid] : -1;
  }
  attn_sync();
  // this split's key range [k_lo, k_hi) (64-key tiles shared evenly)
  int maxp0 = -1, wmin = INT_MAX;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    maxp0 = max(maxp0, qpos[j]);
    if (qpos[j] >= 0) wmin = min(wmin, qpos[j]);
  }
  const int* wpos = sh.wpos;
  const int tiles_all = (maxp0 + 1 + kTcKT - 1) / kTcKT;
  const int t_lo = (int)((long)split * tiles_all / n_splits), t_hi = (int)((long)(split + 1) * tiles_all / n_splits);
  const int k_lo = t_lo * kTcKT, k_hi = min(t_hi * kTcKT, maxp0 + 1);
  const int n_keys = k_hi;
  const int n_tiles = t_hi;  // tiles [t_lo, t_hi) of this split

  // Tile `tile` -> ring stage (tile - t_lo) % STAGES.  `hist`: skip this
  // forward's window rows (the append below writes them straight into the
  // stage), so every resident tile -- window tile included -- can be requested
  // before the programmatic-dependency wait.
  auto issue = [&](int tile, bool hist) {
    if (tile < n_tiles) {
      uint8_t* st = ring + ((tile - t_lo) % kTcStages) * (uint32_t)SM::stage;
      constexpr int CPR = HD / 8;         // 16-byte chunks per row
      constexpr int RPP = 128 / CPR;      // rows per pass
      const int c = (tid % CPR) * 8, r0 = tid / CPR;
      __nv_bfloat16* Kd = reinterpret_cast<__nv_bfloat16*>(st) + r0 * RS + c;
      __nv_bfloat16* Vd = reinterpret_cast<__nv_bfloat16*>(st + SM::tile) + r0 * RS + c;
      const int k0 = tile * kTcKT + r0;
      const __nv_bfloat16* ks = kslab + (size_t)k0 * HD + c;
      const __nv_bfloat16* vs = vslab + (size_t)k0 * HD + c;
      const bool check = hist && tile * kTcKT + kTcKT > wmin;  // tile holds window rows
#pragma unroll
      for (int j = 0; j < kTcKT / RPP; ++j) {
        const int key = k0 + j * RPP;
        if (key < n_keys) {
          bool win = false;
          if (check && key >= wmin)
            for (int q = 0; q < q_len; ++q) win |= wpos[q] == key;
          if (!win) {
            // (plain cp.async: the L2::cache_hint evict-first variant raised illegal-instruction faults
            // in the templated decode kernel as it did in wide-GQA block mode before)
            cp_async16(Kd + j * RPP * RS, ks + (size_t)j * RPP * HD);
            cp_async16(Vd + j * RPP * RS, vs + (size_t)j * RPP * HD);
          }
        } else {  // rows past the context: zeros (P is 0 there, and 0 * stale NaN would poison P.V)
          *reinterpret_cast<uint4*>(Kd + j * RPP * RS) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(Vd + j * RPP * RS) = make_uint4(0, 0, 0, 0);
        }
      }
    }
    cp_async_commit();  // always commit (possibly empty) to keep group counting uniform
  };
  // The first STAGES tiles (KV history; the cache rows of this layer were last
  // written >= 2 launches back) start loading now, overlapping the tail of the
  // qkv GEMM.
  // (prefill blocks: the preceding rope_append wrote these rows -- after the wait)
  if (!blk)
    for (int i = 0; i < kTcStages; ++i) issue(t_lo + i, true);

  if (pdl) {
    griddep_wait();
    griddep_launch();
  }
  if (A.trace && tid == 0) A.tr_t[1] = gtime();
  if (blk)
    for (int i = 0; i < kTcStages; ++i) issue(t_lo + i, false);
  {
    // One pass, one round trip: thread -> (row j, 8 rotary pairs from c8).  Q
    // rows j < 16 are rotated into Qs (zero past nQ); window tokens j < q_len
    // have K rotated and K / V appended to the cache and, for resident tiles,
    // to their ring stage.  All global loads are issued before any use.
    constexpr int CPW = HALF / 8;
    const int j = tid / CPW, c8 = (tid % CPW) * 8;
    uint4 qx0 = make_uint4(0, 0, 0, 0), qx1 = qx0, kx0 = qx0, kx1 = qx0, vx0 = qx0, vx1 = qx0;
    float4 qc0{}, qc1{}, qs0{}, qs1{}, kc0{}, kc1{}, ks0{}, ks1{};
    const bool qv = j < 16 && j < nQ;
    if (qv && blk) {
      const __nv_bfloat16* src = A.qr + ((size_t)(seq * q_len + qtok[j]) * nq + qhead[j]) * HD + c8;
      qx0 = *reinterpret_cast<const uint4*>(src);
      qx1 = *reinterpret_cast<const uint4*>(src + HALF);
    } else if (qv) {
      const int p = qpos[j];
      const int pc = p < 0 ? 0 : (p >= max_pos ? max_pos - 1 : p);
      const __nv_bfloat16* src = seq_rows + (size_t)qtok[j] * row_w + qhead[j] * HD + c8;
      qx0 = *reinterpret_cast<const uint4*>(src);
      qx1 = *reinterpret_cast<const uint4*>(src + HALF);
      const float4* cp = reinterpret_cast<const float4*>(cosT + (size_t)pc * HALF + c8);
      const float4* sp4 = reinterpret_cast<const float4*>(sinT + (size_t)pc * HALF + c8);
      qc0 = cp[0], qc1 = cp[1], qs0 = sp4[0], qs1 = sp4[1];
    }
    const int pk = !blk && j < q_len ? wpos[j] : -1;
    const bool kv = pk >= k_lo && pk < k_hi;  // (pk < 0: padding, never in range)
    if (kv) {
      const int pc = pk >= max_pos ? max_pos - 1 : pk;
      const __nv_bfloat16* src = seq_rows + (size_t)j * row_w + (nq + kvh) * HD + c8;
      kx0 = *reinterpret_cast<const uint4*>(src);
      kx1 = *reinterpret_cast<const uint4*>(src + HALF);
      const __nv_bfloat16* vsrc = seq_rows + (size_t)j * row_w + (nq + nkv + kvh) * HD + c8;
      vx0 = *reinterpret_cast<const uint4*>(vsrc);
      vx1 = *reinterpret_cast<const uint4*>(vsrc + HALF);
      const float4* cp = reinterpret_cast<const float4*>(cosT + (size_t)pc * HALF + c8);
      const float4* sp4 = reinterpret_cast<const float4*>(sinT + (size_t)pc * HALF + c8);
      kc0 = cp[0], kc1 = cp[1], ks0 = sp4[0], ks1 = sp4[1];
    }
    // (x0, x1) pairs -> (x0 c - x1 s, x1 c + x0 s), bf16
    auto rot = [](uint4 x0, uint4 x1, float4 c0, float4 c1, float4 s0, float4 s1, uint4& a, uint4& b) {
      const __nv_bfloat16* u = reinterpret_cast<const __nv_bfloat16*>(&x0);
      const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(&x1);
      const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      const float ss[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      __nv_bfloat16* pa = reinterpret_cast<__nv_bfloat16*>(&a);
      __nv_bfloat16* pb = reinterpret_cast<__nv_bfloat16*>(&b);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float f0 = __bfloat162float(u[i]), f1 = __bfloat162float(w[i]);
        pa[i] = __float2bfloat16_rn(f0 * cc[i] - f1 * ss[i]);
        pb[i] = __float2bfloat16_rn(f1 * cc[i] + f0 * ss[i]);
      }
    };
    if (j < 16) {
      uint4 a = make_uint4(0, 0, 0, 0), b2 = a;
      if (qv && blk) a = qx0, b2 = qx1;
      else if (qv) rot(qx0, qx1, qc0, qc1, qs0, qs1, a, b2);
      *reinterpret_cast<uint4*>(Qs + j * RS + c8) = a;
      *reinterpret_cast<uint4*>(Qs + j * RS + HALF + c8) = b2;
    }
    if (kv) {
      uint4 a, b2;
      rot(kx0, kx1, kc0, kc1, ks0, ks1, a, b2);
      *reinterpret_cast<uint4*>(kslab + (size_t)pk * HD + c8) = a;
      *reinterpret_cast<uint4*>(kslab + (size_t)pk * HD + HALF + c8) = b2;
      *reinterpret_cast<uint4*>(vslab + (size_t)pk * HD + c8) = vx0;
      *reinterpret_cast<uint4*>(vslab + (size_t)pk * HD + HALF + c8) = vx1;
      const int ti = pk / kTcKT - t_lo;
      if (ti < kTcStages) {
        const int r = pk - (pk / kTcKT) * kTcKT;
        __nv_bfloat16* Kd = reinterpret_cast<__nv_bfloat16*>(ring + ti * (uint32_t)SM::stage) + r * RS;
        __nv_bfloat16* Vd = reinterpret_cast<__nv_bfloat16*>(ring + ti * (uint32_t)SM::stage + SM::tile) + r * RS;
        *reinterpret_cast<uint4*>(Kd + c8) = a;
        *reinterpret_cast<uint4*>(Kd + HALF + c8) = b2;
        *reinterpret_cast<uint4*>(Vd + c8) = vx0;
        *reinterpret_cast<uint4*>(Vd + HALF + c8) = vx1;
      }
    }
  }
  __threadfence_block();
  attn_sync();
  if (A.trace && tid == 0) A.tr_t[2] = gtime();

  // Q fragments (A operand), loaded once
  const uint32_t qs_base = (uint32_t)__cvta_generic_to_shared(Qs);
  uint32_t qa[KSTEP][4];
  {
    const int mi = lane >> 3, ri = lane & 7;
    const int row = ri + (mi & 1) * 8;
#pragma unroll
    for (int ks = 0; ks < KSTEP; ++ks) {
      int col = ks * 16 + (mi >> 1) * 8;
      ldsm_x4(qs_base + (uint32_t)(row * RS + col) * 2, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
  }
  const int g = lane >> 2, t4 = lane & 3;
  const int pos_lo = qpos[g], pos_hi = qpos[g + 8];
  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

  for (int tile = t_lo; tile < n_tiles; ++tile) {
    cp_async_wait<kTcStages - 1>();
    attn_sync();
    const uint8_t* st = ring + ((tile - t_lo) % kTcStages) * (uint32_t)SM::stage;
    const uint32_t kb = (uint32_t)__cvta_generic_to_shared(st);
    const uint32_t vb = kb + (uint32_t)SM::tile;
    const int kw = warp * 16;  // this warp's 16 keys within the tile
    // S = Q K^T for keys kw..kw+15 (two n8 tiles)
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
    // mask + scale, online softmax (rows g and g+8)
    const int kbase = tile * kTcKT + kw + 2 * t4;
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
    float p[8], sum_lo = 0.f, sum_hi = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      p[i] = (mn_lo == -INFINITY) ? 0.f : __expf(v[i] - mn_lo);
      p[4 + i] = (mn_hi == -INFINITY) ? 0.f : __expf(v[4 + i] - mn_hi);
      sum_lo += p[i];
      sum_hi += p[4 + i];
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
    // P (A operand, k = the warp's 16 keys) straight from the S accumulators
    const uint32_t pa0 = pack_bf16(p[0], p[1]), pa1 = pack_bf16(p[4], p[5]);
    const uint32_t pa2 = pack_bf16(p[2], p[3]), pa3 = pack_bf16(p[6], p[7]);
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
    attn_sync();  // this stage is free: refill it (tiles past the resident ones read the appended cache)
    issue(tile + kTcStages, false);
  }
  cp_async_wait<0>();
  attn_sync();
  if (A.trace && tid == 0) A.tr_t[3] = gtime();
  // combine the 4 warps in order (smem partials alias the drained ring)
  float* comb = reinterpret_cast<float*>(ring);
  float* cm = comb + 4 * 16 * HD;
  float* cl = cm + 4 * 16;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    int d = n * 8 + 2 * t4;
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
  attn_sync();
  if (!SPLIT || n_splits == 1) {
    // 8 consecutive dims per thread: one 16-byte streaming store (scalar 2-byte stores of the output
    // row cost ~2 us under the weight stream, like the GEMM epilogue's)
    for (int e = tid; e < nQ * (HD / 8); e += 128) {
      const int j = e / (HD / 8), d0 = (e % (HD / 8)) * 8;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, cm[w * 16 + j]);
      float f[4], L = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float mw = cm[w * 16 + j];
        f[w] = (mw == -INFINITY) ? 0.f : __expf(mw - M);
        L += cl[w * 16 + j] * f[w];
      }
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc[i] = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[i] += comb[(w * 16 + j) * HD + d0 + i] * f[w];
      }
      uint4 pk;
      uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        pw[i] = pack_bf16(L > 0.f ? acc[2 * i] / L : 0.f, L > 0.f ? acc[2 * i + 1] / L : 0.f);
      __stcs(reinterpret_cast<uint4*>(out + ((size_t)(seq * q_len + qtok[j]) * nq + qhead[j]) * HD + d0), pk);
    }
    return;
  }
  // ---- split partial: warps merged in order, unnormalised
  const size_t item = (size_t)seq * nkv + kvh;
  float* mypart = sp.part + (item * n_splits + split) * 16 * HD;
  float* myml = sp.ml + (item * n_splits + split) * 16 * 2;
  for (int e = tid; e < nQ * HD; e += 128) {
    int j = e / HD, d = e % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, cm[w * 16 + j]);
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      float mw = cm[w * 16 + j];
      float f = (mw == -INFINITY) ? 0.f : __expf(mw - M);
      L += cl[w * 16 + j] * f;
      acc += comb[(w * 16 + j) * HD + d] * f;
    }
    __stcg(mypart + j * HD + d, acc);
    if (d == 0) {
      __stcg(myml + j * 2, M);
      __stcg(myml + j * 2 + 1, L);
    }
  }
  __threadfence();
  attn_sync();
  if (tid == 0) sh.last = atomicAdd(sp.counter + item, 1) == n_splits - 1;
  attn_sync();
  if (!sh.last) return;
  __threadfence();
  for (int e = tid; e < nQ * HD; e += 128) {
    int j = e / HD, d = e % HD;
    float M = -INFINITY;
    for (int z = 0; z < n_splits; ++z) M = fmaxf(M, __ldcg(sp.ml + ((item * n_splits + z) * 16 + j) * 2));
    float L = 0.f, acc = 0.f;
    for (int z = 0; z < n_splits; ++z) {
      const float mz = __ldcg(sp.ml + ((item * n_splits + z) * 16 + j) * 2);
      const float f = (mz == -INFINITY) ? 0.f : __expf(mz - M);
      L += __ldcg(sp.ml + ((item * n_splits + z) * 16 + j) * 2 + 1) * f;
      acc += __ldcg(sp.part + ((item * n_splits + z) * 16 + j) * HD + d) * f;
    }
    out[((size_t)(seq * q_len + qtok[j]) * nq + qhead[j]) * HD + d] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
  }
  if (tid == 0) sp.counter[item] = 0;  // ready for the next launch
}


}  // namespace sb
