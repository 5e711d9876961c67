// The draft loop of one speculative iteration as ONE persistent kernel (K1):
// k autoregressive steps of the small draft model for b sequences, greedy.
//
// The draft (LLaMA-68M: 2 layers, h 768) is latency-bound: ~13 kernel
// launches per step at ~5 us each against a ~13 us HBM floor.  Here one CTA
// per SM runs every step:
//
//   per step j = 1..k (step 1 re-feeds the last two committed tokens, q = 2)
//     per layer:  qkv (fused 1/rms, RoPE, KV append) | attention | o (+resid)
//                 | gate/up (silu*up) | down (+resid)
//     lm_head (fused argmax partials) | finalize (token -> next step's input)
//
// separated by grid barriers.  The GEMMs are ROW-PARALLEL: a warp owns whole
// 16-row (or one-head) output units over the full K (mma.sync m16n8k16, bf16
// in / fp32 accumulate, weights streamed through a per-warp 3-stage cp.async
// ring) -- no split-K, so no cross-CTA fix-up chain at phase ends (the lesson
// of persistent.cu).  Every CTA rebuilds the (<= 16-token) GEMM input in
// shared memory itself (raw bf16 residual; 1/rms applied to the accumulator,
// the engine's fused-norm contract), so norms need no extra barrier.
//
// Outputs follow the token-sink protocol of sb_decoder_forward_ex:
//   v_ids[s*(k+1) + j] = d_j,  ds_ids[s] = d_j,  ds_pos[s] = d_base[s] + j.
#include <climits>
#include <cstring>

#include "common.cuh"
#include "grid_sync.cuh"
#include "kernels.cuh"
#include "mma_ptx.cuh"

namespace sb {

constexpr int DL_THREADS = 256;
constexpr int DL_WARPS = 8;
constexpr int DL_MAXT = 16;    // tokens per step (2b in step 1)
constexpr int DL_MAXL = 16;    // draft layers
constexpr int DL_KC = 64;      // k per W stage
constexpr int DL_WRS = DL_KC + 8;
constexpr int DL_WSTAGES = 5;
constexpr int DL_WSTAGE = 16 * DL_WRS * 2;

struct DlParams {
  int L, H, nq, nkv, hd, ffn, V, max_pos, ctx_max, b, k, G, x_cap;
  float eps, att_scale;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* lm_head;
  const __nv_bfloat16* w_qkv[DL_MAXL];
  const __nv_bfloat16* w_o[DL_MAXL];
  const __nv_bfloat16* w_gu[DL_MAXL];
  const __nv_bfloat16* w_down[DL_MAXL];
  const float* cosT;
  const float* sinT;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  size_t layer_kv;
  const int32_t* d1_ids;
  const int32_t* d1_pos;
  const int32_t* slot;
  const int32_t* d_base;
  int32_t* v_ids;
  int32_t* ds_ids;
  int32_t* ds_pos;
  float* resid;          // [T][H]
  __nv_bfloat16* qr;     // [T][nq*hd]
  __nv_bfloat16* att;    // [T][nq*hd]
  __nv_bfloat16* act;    // [T][ffn]
  float* am_val;         // [G*8][b]
  int* am_idx;
  unsigned* sync;        // [0] barrier, [1] exit
  unsigned long long* trace;  // diagnostics: globaltimer at every barrier (CTA 0), NULL = off
};

struct DlTok {
  int T, q;
  int id[DL_MAXT], pos[DL_MAXT];
};

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(ok ? 16 : 0)
               : "memory");
}

// 16 weight rows [r0, r0+16) of W [N][K] times the (<= 16) tokens in X smem
// [16][XS]: acc[nt] = rows x tokens nt*8..nt*8+7 (mma C layout).
__device__ __forceinline__ void warp_gemm16(const __nv_bfloat16* __restrict__ W, int N, int K, int r0, uint32_t xs,
                                            int XS, uint8_t* wst, float (&acc)[2][4], int c_lo = 0, int c_hi = -1) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int n = 0; n < 2; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
  const int nch = c_hi < 0 ? K / DL_KC : c_hi;
  auto issue = [&](int c) {
    if (c < nch) {
      uint8_t* st = wst + (c % DL_WSTAGES) * DL_WSTAGE;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int pce = lane + 32 * i, row = pce >> 3, c16 = pce & 7;
        const bool ok = r0 + row < N;
        cp_async16_zfill(st + (row * DL_WRS + c16 * 8) * 2, W + (size_t)(ok ? r0 + row : 0) * K + c * DL_KC + c16 * 8,
                         ok);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int i = 0; i < DL_WSTAGES - 1; ++i) issue(c_lo + i);
  const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(wst);
  for (int c = c_lo; c < nch; ++c) {
    issue(c + DL_WSTAGES - 1);
    cp_async_wait<DL_WSTAGES - 1>();
    __syncwarp();
    const uint32_t sa = wbase + (uint32_t)((c % DL_WSTAGES) * DL_WSTAGE);
#pragma unroll
    for (int ks = 0; ks < DL_KC / 16; ++ks) {
      uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
      ldsm_x4(sa + (uint32_t)(((lane & 15) * DL_WRS + ks * 16 + (lane >> 4) * 8) * 2), a0, a1, a2, a3);
      const int tok = (lane & 7) + (lane >> 4) * 8;
      ldsm_x4(xs + (uint32_t)((tok * XS + c * DL_KC + ks * 16 + ((lane >> 3) & 1) * 8) * 2), b0, b1, b2, b3);
      mma_bf16(acc[0], a0, a1, a2, a3, b0, b1);
      mma_bf16(acc[1], a0, a1, a2, a3, b2, b3);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  __syncwarp();
}

// All 8 warps of the CTA on one unit of mt 16-row tiles: warp w takes k-chunks
// [w*nch/8, (w+1)*nch/8) of every tile; partials meet in shared memory (over
// the drained W stages) and warp 0 sums them in warp order into `acc`.
// (Small matrices have too few 16-row units to keep 148 x 8 warps streaming.)
template <int MT>
__device__ __forceinline__ void cta_gemm_unit(const __nv_bfloat16* __restrict__ W, int N, int K, int r0, int mt,
                                              uint32_t xs, int XS, uint8_t* wst_all, float (&acc)[MT][2][4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = K / DL_KC;
  const int c_lo = warp * nch / DL_WARPS, c_hi = (warp + 1) * nch / DL_WARPS;
  uint8_t* wst = wst_all + warp * DL_WSTAGES * DL_WSTAGE;
#pragma unroll
  for (int a = 0; a < MT; ++a) {
    if (a >= mt) continue;
    if (c_lo < c_hi) {
      warp_gemm16(W, N, K, r0 + a * 16, xs, XS, wst, acc[a], c_lo, c_hi);
    } else {
      acc[a][0][0] = acc[a][0][1] = acc[a][0][2] = acc[a][0][3] = 0.f;
      acc[a][1][0] = acc[a][1][1] = acc[a][1][2] = acc[a][1][3] = 0.f;
    }
  }
  __syncthreads();  // every warp's ring drained: reuse it as the reduction buffer
  float* red = reinterpret_cast<float*>(wst_all);
#pragma unroll
  for (int a = 0; a < MT; ++a)
    if (a < mt)
#pragma unroll
      for (int i = 0; i < 8; ++i) red[((warp * MT + a) * 8 + i) * 32 + lane] = acc[a][i >> 2][i & 3];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int a = 0; a < MT; ++a)
      if (a < mt)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float v = 0.f;
          for (int w = 0; w < DL_WARPS; ++w) v += red[((w * MT + a) * 8 + i) * 32 + lane];
          acc[a][i >> 2][i & 3] = v;
        }
  }
  __syncthreads();
}

// grid barrier: every CTA arrives once per phase
__device__ __forceinline__ void dl_barrier(const DlParams& p, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[epoch] = globaltimer();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p.sync, 1u);
    wait_geq(p.sync, epoch * (unsigned)p.G);
    __threadfence();
  }
  __syncthreads();
}

// X smem [16][XS] = bf16(raw source rows) (rows >= T zero) and inv[t] = 1/rms.
// Sources: fp32 residual rows `src[rows[t]]`, or (layer 0) the bf16 embedding
// rows of the step's tokens.  16-byte loads, a batch of 8 in flight per thread.
__device__ void dl_load_x(const DlParams& p, const DlTok& tk, int layer0_embed, const float* src, int K, int ld,
                          __nv_bfloat16* xs, int XS, float* inv, bool norm, const int* rows, int T) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c8 = K / 8;  // 8-element chunks per row
  const int total = DL_MAXT * c8;
  for (int e0 = tid; e0 < total; e0 += DL_THREADS * 8) {
    float v[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = e0 + i * DL_THREADS;
      const int t = e / c8, c = (e % c8) * 8;
#pragma unroll
      for (int z = 0; z < 8; ++z) v[i][z] = 0.f;
      if (e >= total || t >= T) continue;
      const int r = rows[t];
      if (layer0_embed) {
        const int id = tk.id[r];
        if (tk.pos[r] < 0 || id < 0 || id >= p.V) continue;
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(p.embed + (size_t)id * p.H + c));
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          const float2 f = __bfloat1622float2(b2[z]);
          v[i][2 * z] = f.x;
          v[i][2 * z + 1] = f.y;
        }
      } else {
        const float4 a4 = __ldcg(reinterpret_cast<const float4*>(src + (size_t)r * ld + c));
        const float4 b4 = __ldcg(reinterpret_cast<const float4*>(src + (size_t)r * ld + c + 4));
        v[i][0] = a4.x, v[i][1] = a4.y, v[i][2] = a4.z, v[i][3] = a4.w;
        v[i][4] = b4.x, v[i][5] = b4.y, v[i][6] = b4.z, v[i][7] = b4.w;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = e0 + i * DL_THREADS;
      if (e >= total) continue;
      const int t = e / c8, c = (e % c8) * 8;
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int z = 0; z < 4; ++z) o2[z] = __floats2bfloat162_rn(v[i][2 * z], v[i][2 * z + 1]);
      *reinterpret_cast<uint4*>(xs + t * XS + c) = o;
    }
  }
  if (!norm) return;
  __syncthreads();
  for (int t = warp; t < DL_MAXT; t += DL_WARPS) {  // 1/rms from the (exact, fp32) sources
    float ss = 0.f;
    if (t < T) {
      const int r = rows[t];
      for (int k = lane * 4; k < K; k += 128) {
        float4 a4;
        if (layer0_embed) {
          const int id = tk.id[r];
          const bool pad = tk.pos[r] < 0 || id < 0 || id >= p.V;
          const uint2 u = pad ? make_uint2(0, 0) : __ldg(reinterpret_cast<const uint2*>(p.embed + (size_t)id * p.H + k));
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
          const float2 f0 = __bfloat1622float2(b2[0]), f1 = __bfloat1622float2(b2[1]);
          a4 = make_float4(f0.x, f0.y, f1.x, f1.y);
        } else {
          a4 = __ldcg(reinterpret_cast<const float4*>(src + (size_t)r * ld + k));
        }
        ss += a4.x * a4.x + a4.y * a4.y + a4.z * a4.z + a4.w * a4.w;
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) inv[t] = t < T ? rsqrtf(ss / (float)K + p.eps) : 0.f;
  }
}

// bf16 activation rows -> X smem (no norm), 8 x 16-byte loads in flight per thread
__device__ void dl_load_xb(const __nv_bfloat16* src, int K, int T, __nv_bfloat16* xs, int XS) {
  const int c8 = K / 8, total = DL_MAXT * c8;
  for (int e0 = threadIdx.x; e0 < total; e0 += DL_THREADS * 8) {
    uint4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = e0 + i * DL_THREADS;
      const int t = e / c8, c = (e % c8) * 8;
      v[i] = (e < total && t < T) ? __ldcg(reinterpret_cast<const uint4*>(src + (size_t)t * K + c)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = e0 + i * DL_THREADS;
      if (e < total) *reinterpret_cast<uint4*>(xs + (e / c8) * XS + (e % c8) * 8) = v[i];
    }
  }
}

__global__ void __launch_bounds__(DL_THREADS, 1) draft_loop_kernel(const __grid_constant__ DlParams p) {
  extern __shared__ __align__(128) uint8_t dsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, c = blockIdx.x;
  const int gw = c * DL_WARPS + warp, GW = p.G * DL_WARPS;
  const int XS = p.x_cap + 8;
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(dsm);
  uint8_t* wst_all = dsm + (size_t)DL_MAXT * XS * 2;
  uint8_t* wst = wst_all + warp * DL_WSTAGES * DL_WSTAGE;
  __shared__ float inv[DL_MAXT];
  __shared__ DlTok tk;
  __shared__ int rows_all[DL_MAXT], rows_last[DL_MAXT];
  __shared__ float rope_c[DL_MAXT * 64], rope_s[DL_MAXT * 64];  // [t][hd/2] at each token's position
  const uint32_t xs_u = (uint32_t)__cvta_generic_to_shared(xs);
  const int H = p.H, hd = p.hd, qd = p.nq * hd, kd = p.nkv * hd;
  griddep_wait();
  unsigned epoch = 0;
  if (p.trace && c == 0 && tid == 0) p.trace[0] = globaltimer();

  for (int j = 1; j <= p.k; ++j) {
    // ---- this step's tokens (step 1: the last two committed tokens per sequence)
    if (tid == 0) {
      tk.q = j == 1 ? 2 : 1;
      tk.T = p.b * tk.q;
      for (int t = 0; t < tk.T; ++t) {
        const int s = t / tk.q, i = t % tk.q;
        tk.id[t] = j == 1 ? p.d1_ids[2 * s + i] : p.ds_ids[s];
        tk.pos[t] = j == 1 ? p.d1_pos[2 * s + i] : p.ds_pos[s];
      }
    }
    if (tid < DL_MAXT) {
      rows_all[tid] = tid;
      rows_last[tid] = tid * (j == 1 ? 2 : 1) + (j == 1 ? 1 : 0);
    }
    __syncthreads();
    const int T = tk.T, q = tk.q;
    for (int e = tid; e < T * (hd / 2); e += DL_THREADS) {
      const int t = e / (hd / 2), i = e % (hd / 2);
      const int ps = tk.pos[t];
      const int pc = ps < 0 ? 0 : (ps >= p.max_pos ? p.max_pos - 1 : ps);
      rope_c[t * 64 + i] = p.cosT[(size_t)pc * (hd / 2) + i];
      rope_s[t * 64 + i] = p.sinT[(size_t)pc * (hd / 2) + i];
    }

    for (int l = 0; l < p.L; ++l) {
      __nv_bfloat16* kcl = p.kc + (size_t)l * p.layer_kv;
      __nv_bfloat16* vcl = p.vc + (size_t)l * p.layer_kv;
      // ======== qkv: one head per unit (RoPE pairs stay lane-local), KV append
      dl_load_x(p, tk, l == 0, p.resid, H, H, xs, XS, inv, true, rows_all, T);
      __syncthreads();
      {
        const int n_units = p.nq + 2 * p.nkv;
        const int mt = hd / 16;
        for (int u = c; u < n_units; u += p.G) {  // one head per CTA, K split over its 8 warps
          float acc[8][2][4];
          cta_gemm_unit<8>(p.w_qkv[l], qd + 2 * kd, H, u * hd, mt, xs_u, XS, wst_all, acc);
          if (warp != 0) continue;
          const int region = u < p.nq ? 0 : (u < p.nq + p.nkv ? 1 : 2);
          const int head = region == 0 ? u : (region == 1 ? u - p.nq : u - p.nq - p.nkv);
          const int g = lane >> 2, t4 = lane & 3, half = hd / 2;
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            if (a >= mt) continue;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int d = a * 16 + g + (e >> 1) * 8;
                const int t = nt * 8 + 2 * t4 + (e & 1);
                if (t >= T) continue;
                const float x = bf16r(acc[a][nt][e] * inv[t]);
                const int ps = tk.pos[t];
                const int s = t / q;
                if (region == 2) {
                  if (ps >= 0)
                    vcl[(((size_t)p.slot[s] * p.nkv + head) * p.ctx_max + ps) * hd + d] = __float2bfloat16_rn(x);
                  continue;
                }
                // partner row d +- hd/2: m-tile a +- hd/32, same lane and element
                const int pa = d < half ? a + hd / 32 : a - hd / 32;
                float xp = 0.f;
#pragma unroll
                for (int aa = 0; aa < 8; ++aa)
                  if (aa == pa) xp = bf16r(acc[aa][nt][e] * inv[t]);
                const int di = d < half ? d : d - half;
                const float cs = rope_c[t * 64 + di], sn = rope_s[t * 64 + di];
                const __nv_bfloat16 ob = __float2bfloat16_rn(d < half ? x * cs - xp * sn : x * cs + xp * sn);
                if (region == 0)
                  p.qr[(size_t)t * qd + head * hd + d] = ob;
                else if (ps >= 0)
                  kcl[(((size_t)p.slot[s] * p.nkv + head) * p.ctx_max + ps) * hd + d] = ob;
              }
          }
        }
      }
      dl_barrier(p, epoch);
      // ======== attention: one warp per (token, q head), lane-per-key for the
      // scores AND for P.V (each lane accumulates its own keys' V rows with
      // 16-byte loads, all in flight); the 32 lane partials meet in shared
      // memory (the idle W-stage area) and each lane sums its output dims.
      {
        const int group = p.nq / p.nkv;
        const int items = T * p.nq;
        float* opart = reinterpret_cast<float*>(wst_all) + warp * 32 * 65;  // [32 lanes][64 dims + pad]
        for (int it = gw; it < items; it += GW) {
          const int t = it / p.nq, h = it % p.nq, s = t / q, kvh = h / group;
          const int ps = tk.pos[t];
          if (ps < 0) continue;
          const __nv_bfloat16* ks = kcl + ((size_t)p.slot[s] * p.nkv + kvh) * p.ctx_max * hd;
          const __nv_bfloat16* vs = vcl + ((size_t)p.slot[s] * p.nkv + kvh) * p.ctx_max * hd;
          const __nv_bfloat16* qv = p.qr + (size_t)t * qd + h * hd;
          const int nk = ps + 1;
          float sc[9];
          float mx = -INFINITY;
#pragma unroll
          for (int m = 0; m < 9; ++m) {
            const int key = lane + 32 * m;
            float dot = -INFINITY;
            if (key < nk) {
              dot = 0.f;
              for (int d0 = 0; d0 < hd; d0 += 8) {
                const uint4 kv4 = __ldcg(reinterpret_cast<const uint4*>(ks + (size_t)key * hd + d0));
                const uint4 qv4 = __ldcg(reinterpret_cast<const uint4*>(qv + d0));
                const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv4);
                const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&qv4);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float2 kf = __bfloat1622float2(k2[i]), qf = __bfloat1622float2(q2[i]);
                  dot = fmaf(qf.x, kf.x, fmaf(qf.y, kf.y, dot));
                }
              }
              dot *= p.att_scale;
            }
            sc[m] = dot;
            mx = fmaxf(mx, dot);
          }
          mx = warp_max(mx);
          float sum = 0.f;
#pragma unroll
          for (int m = 0; m < 9; ++m) {
            sc[m] = (lane + 32 * m < nk) ? __expf(sc[m] - mx) : 0.f;
            sum += sc[m];
          }
          sum = warp_sum(sum);
          const float rs = sum > 0.f ? 1.f / sum : 0.f;
          for (int d0 = 0; d0 < hd; d0 += 64) {  // 64 output dims per pass
            float o[64];
#pragma unroll
            for (int e = 0; e < 64; ++e) o[e] = 0.f;
#pragma unroll
            for (int m = 0; m < 9; ++m) {
              const int key = lane + 32 * m;
              if (key < nk) {
#pragma unroll
                for (int c8 = 0; c8 < 8; ++c8) {
                  const uint4 v4 = __ldcg(reinterpret_cast<const uint4*>(vs + (size_t)key * hd + d0 + c8 * 8));
                  const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&v4);
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const float2 vf = __bfloat1622float2(v2[i]);
                    o[c8 * 8 + 2 * i] = fmaf(sc[m], vf.x, o[c8 * 8 + 2 * i]);
                    o[c8 * 8 + 2 * i + 1] = fmaf(sc[m], vf.y, o[c8 * 8 + 2 * i + 1]);
                  }
                }
              }
            }
#pragma unroll
            for (int e = 0; e < 64; ++e) opart[lane * 65 + e] = o[e];
            __syncwarp();
            for (int e = lane; e < 64; e += 32) {
              float acc = 0.f;
              for (int l2 = 0; l2 < 32; ++l2) acc += opart[l2 * 65 + e];
              p.att[(size_t)t * qd + h * hd + d0 + e] = __float2bfloat16_rn(acc * rs);
            }
            __syncwarp();
          }
        }
      }
      dl_barrier(p, epoch);
      // ======== o: 16-row units, + residual (layer 0: the embedding)
      dl_load_xb(p.att, qd, T, xs, XS);
      __syncthreads();
      for (int u = c; u * 16 < H; u += p.G) {
        float acc1[1][2][4];
        cta_gemm_unit<1>(p.w_o[l], H, qd, u * 16, 1, xs_u, XS, wst_all, acc1);
        if (warp != 0) continue;
        float(&acc)[2][4] = acc1[0];
        const int g = lane >> 2, t4 = lane & 3;
        float prev[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {  // all residual (layer 0: embedding) loads first
            const int n = u * 16 + g + (e >> 1) * 8, t = nt * 8 + 2 * t4 + (e & 1);
            prev[nt][e] = 0.f;
            if (t >= T || n >= H) continue;
            if (l == 0) {
              const int id = tk.id[t];
              const bool pad = tk.pos[t] < 0 || id < 0 || id >= p.V;
              prev[nt][e] = pad ? 0.f : __bfloat162float(p.embed[(size_t)id * H + n]);
            } else {
              prev[nt][e] = __ldcg(p.resid + (size_t)t * H + n);
            }
          }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = u * 16 + g + (e >> 1) * 8, t = nt * 8 + 2 * t4 + (e & 1);
            if (t < T && n < H) p.resid[(size_t)t * H + n] = prev[nt][e] + acc[nt][e];
          }
      }
      dl_barrier(p, epoch);
      // ======== gate/up (interleaved rows): silu(g) * u
      dl_load_x(p, tk, 0, p.resid, H, H, xs, XS, inv, true, rows_all, T);
      __syncthreads();
      for (int u = gw; u * 16 < 2 * p.ffn; u += GW) {
        float acc[2][4];
        warp_gemm16(p.w_gu[l], 2 * p.ffn, H, u * 16, xs_u, XS, wst, acc);
        const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = u * 16 + g + (e >> 1) * 8, t = nt * 8 + 2 * t4 + (e & 1);
            const float x = t < T ? acc[nt][e] * inv[t] : 0.f;
            const float other = __shfl_xor_sync(0xffffffffu, x, 4);  // row g^1 (gate/up pair)
            if (!(g & 1) && t < T && n < 2 * p.ffn)
              p.act[(size_t)t * p.ffn + n / 2] = __float2bfloat16_rn(x / (1.f + __expf(-x)) * other);
          }
      }
      dl_barrier(p, epoch);
      // ======== down: 16-row units over K = ffn, + residual
      dl_load_xb(p.act, p.ffn, T, xs, XS);
      __syncthreads();
      for (int u = c; u * 16 < H; u += p.G) {
        float acc1[1][2][4];
        cta_gemm_unit<1>(p.w_down[l], H, p.ffn, u * 16, 1, xs_u, XS, wst_all, acc1);
        if (warp != 0) continue;
        float(&acc)[2][4] = acc1[0];
        const int g = lane >> 2, t4 = lane & 3;
        float prev[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = u * 16 + g + (e >> 1) * 8, t = nt * 8 + 2 * t4 + (e & 1);
            prev[nt][e] = (t < T && n < H) ? __ldcg(p.resid + (size_t)t * H + n) : 0.f;
          }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = u * 16 + g + (e >> 1) * 8, t = nt * 8 + 2 * t4 + (e & 1);
            if (t < T && n < H) p.resid[(size_t)t * H + n] = prev[nt][e] + acc[nt][e];
          }
      }
      dl_barrier(p, epoch);
    }
    // ======== lm_head on each sequence's last token, fused argmax partials
    dl_load_x(p, tk, p.L == 0, p.resid, H, H, xs, XS, inv, true, rows_last, p.b);
    __syncthreads();
    {
      float bv[2][2];
      int bi[2][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) bv[nt][0] = bv[nt][1] = -INFINITY, bi[nt][0] = bi[nt][1] = INT_MAX;
      for (int u = gw; u * 16 < p.V; u += GW) {
        float acc[2][4];
        warp_gemm16(p.lm_head, p.V, H, u * 16, xs_u, XS, wst, acc);
        const int g = lane >> 2;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = u * 16 + g + (e >> 1) * 8, tt = e & 1;
            const int t = nt * 8 + 2 * (lane & 3) + tt;
            const float v = (n < p.V && t < p.b) ? acc[nt][e] * inv[t] : -INFINITY;
            ArgMax a = argmax_merge(ArgMax{bv[nt][tt], bi[nt][tt]}, ArgMax{v, n < p.V ? n : INT_MAX});
            bv[nt][tt] = a.v;
            bi[nt][tt] = a.i;
          }
      }
      // merge the 8 row-groups (lanes with equal lane&3) of the warp
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          ArgMax a{bv[nt][tt], bi[nt][tt]};
#pragma unroll
          for (int o = 4; o < 32; o <<= 1)
            a = argmax_merge(a, ArgMax{__shfl_xor_sync(0xffffffffu, a.v, o), __shfl_xor_sync(0xffffffffu, a.i, o)});
          const int t = nt * 8 + 2 * (lane & 3) + tt;
          if (lane < 4 && t < p.b) {
            p.am_val[(size_t)gw * p.b + t] = a.v;
            p.am_idx[(size_t)gw * p.b + t] = a.i;
          }
        }
    }
    dl_barrier(p, epoch);
    // ======== finalize: sequence s by warp 0 of CTA s
    if (warp == 0 && c < p.b) {
      const int s = c;
      ArgMax a{-INFINITY, INT_MAX};
      for (int w0 = lane; w0 < GW; w0 += 32 * 8) {
        float vv[8];
        int ii[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int w = w0 + 32 * i;
          vv[i] = w < GW ? __ldcg(&p.am_val[(size_t)w * p.b + s]) : -INFINITY;
          ii[i] = w < GW ? __ldcg(&p.am_idx[(size_t)w * p.b + s]) : INT_MAX;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) a = argmax_merge(a, ArgMax{vv[i], ii[i]});
      }
      a = warp_argmax(a);
      if (lane == 0) {
        p.v_ids[(size_t)s * (p.k + 1) + j] = a.i;
        p.ds_ids[s] = a.i;
        p.ds_pos[s] = p.d_base[s] + j;
      }
    }
    dl_barrier(p, epoch);
  }
  griddep_launch();
  // ---- exit: the last CTA out resets the barrier words for the next launch
  if (tid == 0) {
    const unsigned prev = atomicAdd(p.sync + 1, 1u);
    if (prev == (unsigned)p.G - 1) {
      p.sync[0] = 0;
      __threadfence();
      p.sync[1] = 0;
      __threadfence();
    }
  }
}

static unsigned long long* g_dl_trace = nullptr;
int set_draft_loop_trace(void* buf) {
  g_dl_trace = (unsigned long long*)buf;
  return 0;
}

int draft_loop_eligible(const sb_decoder_t* m, int b) {
  if (m->arch != SB_ARCH_LLAMA || m->dtype != SB_BF16 || m->tp) return 0;
  if (2 * b > DL_MAXT || b < 1 || m->n_layers > DL_MAXL) return 0;
  if (m->head_dim != 64 && m->head_dim != 128) return 0;
  if (m->hidden % DL_KC || m->ffn % DL_KC || (m->n_heads * m->head_dim) % DL_KC) return 0;
  return 1;
}

size_t draft_loop_smem(const sb_decoder_t* m) {
  int cap = m->hidden;
  if (m->ffn > cap) cap = m->ffn;
  if (m->n_heads * m->head_dim > cap) cap = m->n_heads * m->head_dim;
  return (size_t)DL_MAXT * (cap + 8) * 2 + (size_t)DL_WARPS * DL_WSTAGES * DL_WSTAGE;
}

int launch_draft_loop(const sb_decoder_t* m, const sb_kvcache_t* kv, int b, int k, const int32_t* d1_ids,
                      const int32_t* d1_pos, const int32_t* slot, const int32_t* d_base, int32_t* v_ids,
                      int32_t* ds_ids, int32_t* ds_pos, const DlBuffers& buf, cudaStream_t st) {
  if (!draft_loop_eligible(m, b) || k < 1) return SB_EUNSUPPORTED;
  DlParams p;
  memset(&p, 0, sizeof(p));
  p.L = m->n_layers;
  p.H = m->hidden;
  p.nq = m->n_heads;
  p.nkv = m->n_kv_heads;
  p.hd = m->head_dim;
  p.ffn = m->ffn;
  p.V = m->vocab;
  p.max_pos = m->max_pos;
  p.ctx_max = kv->ctx_max;
  if (kv->ctx_max > 32 * 9) return SB_EUNSUPPORTED;  // lane-per-key attention holds <= 288 keys
  p.b = b;
  p.k = k;
  p.eps = m->rms_eps;
  p.att_scale = 1.0f / sqrtf((float)m->head_dim);
  int cap = m->hidden;
  if (m->ffn > cap) cap = m->ffn;
  if (m->n_heads * m->head_dim > cap) cap = m->n_heads * m->head_dim;
  p.x_cap = cap;
  static int G = 0;
  if (!G) G = num_sms();
  p.G = G;
  p.embed = (const __nv_bfloat16*)m->embed;
  p.lm_head = (const __nv_bfloat16*)m->lm_head;
  for (int l = 0; l < m->n_layers; ++l) {
    p.w_qkv[l] = (const __nv_bfloat16*)m->w_qkv[l];
    p.w_o[l] = (const __nv_bfloat16*)m->w_o[l];
    p.w_gu[l] = (const __nv_bfloat16*)m->w_gu[l];
    p.w_down[l] = (const __nv_bfloat16*)m->w_down[l];
  }
  p.cosT = m->rope_cos;
  p.sinT = m->rope_sin;
  p.kc = (__nv_bfloat16*)kv->k;
  p.vc = (__nv_bfloat16*)kv->v;
  p.layer_kv = (size_t)kv->slots * m->n_kv_heads * kv->ctx_max * m->head_dim;
  p.d1_ids = d1_ids;
  p.d1_pos = d1_pos;
  p.slot = slot;
  p.d_base = d_base;
  p.v_ids = v_ids;
  p.ds_ids = ds_ids;
  p.ds_pos = ds_pos;
  p.resid = buf.resid;
  p.qr = (__nv_bfloat16*)buf.qr;
  p.att = (__nv_bfloat16*)buf.att;
  p.act = (__nv_bfloat16*)buf.act;
  p.am_val = buf.am_val;
  p.am_idx = buf.am_idx;
  p.sync = buf.sync;
  p.trace = g_dl_trace;
  const size_t smem = draft_loop_smem(m);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(draft_loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    attr = smem;
  }
  return launch_k(draft_loop_kernel, dim3(G), dim3(DL_THREADS), smem, st, p);
}

}  // namespace sb
