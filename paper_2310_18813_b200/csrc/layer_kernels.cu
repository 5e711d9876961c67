// Decoder-layer kernels other than the GEMMs: embedding gather, RMSNorm,
// RoPE + KV append, and KV-cache attention with the causal mask inside the
// speculative window (K3).  All are HBM/latency-bound.
//
// Numerics contract (mirrored by oracle/model_ref.py):
//   residual stream fp32; GEMM inputs rounded to the model dtype; on the bf16
//   path RMSNorm is fused into the GEMMs (input = bf16(residual * gain), written
//   by the residual's producer; output scaled by 1/rms), on the fp32 path the normalised
//   input is materialised (same math); RoPE applied in fp32 from a host-built fp32 cos/sin
//   table then rounded; attention scores/softmax/accumulation in fp32 with a
//   fixed key order (64-key tiles, ascending) so a query's output does not
//   depend on how many other queries share the launch (batch invariance:
//   spec == greedy exactly in fp32 mode).
#include "common.cuh"
#include "kernels.cuh"
#include "mma_ptx.cuh"
#include "attn_tc.cuh"

namespace sb {

thread_local int g_kernel_count = 0;
unsigned long long* g_cta_trace = nullptr;
int g_cta_trace_seq = 0;

// ---------------------------------------------------------------- embedding
template <typename T>
__global__ void embed_kernel(const T* __restrict__ table, const int32_t* __restrict__ ids,
                             const int32_t* __restrict__ pos, float* __restrict__ h, int hidden, int vocab,
                             const T* __restrict__ pos_table, int pos_offset) {
  griddep_wait();
  griddep_launch();
  int t = blockIdx.x;
  int id = ids[t];
  bool pad = pos != nullptr && pos[t] < 0;
  if (id < 0 || id >= vocab) pad = true;
  const T* row = table + (size_t)(pad ? 0 : id) * hidden;
  // OPT: learned absolute positions, row p + offset (the reference model's offset of 2)
  const T* prow = (pos_table && !pad) ? pos_table + (size_t)(pos[t] + pos_offset) * hidden : nullptr;
  float* out = h + (size_t)t * hidden;
  for (int i = threadIdx.x; i < hidden; i += blockDim.x)
    out[i] = pad ? 0.f : (prow ? to_f32(row[i]) + to_f32(prow[i]) : to_f32(row[i]));
}

int launch_embed(int dtype, const void* table, const int32_t* ids, const int32_t* pos, float* h, int n_tok,
                 int hidden, int vocab, cudaStream_t st, const void* pos_table, int pos_offset) {
  if (n_tok <= 0) return 0;
  if (pos_table && !pos) return SB_EINVAL;
  if (dtype == SB_BF16)
    return launch_k(embed_kernel<__nv_bfloat16>, dim3(n_tok), dim3(256), 0, st, (const __nv_bfloat16*)table, ids, pos,
                    h, hidden, vocab, (const __nv_bfloat16*)pos_table, pos_offset);
  return launch_k(embed_kernel<float>, dim3(n_tok), dim3(256), 0, st, (const float*)table, ids, pos, h, hidden, vocab,
                  (const float*)pos_table, pos_offset);
}

// Embedding for the fused-RMSNorm path: fp32 residual, its bf16 copy (the
// next GEMM's X) and the row's sum of squares (one partial per token).
__global__ void __launch_bounds__(256) embed_norm_kernel(const __nv_bfloat16* __restrict__ table,
                                                         const int32_t* __restrict__ ids,
                                                         const int32_t* __restrict__ pos, float* __restrict__ h,
                                                         __nv_bfloat16* __restrict__ xb, float* __restrict__ part,
                                                         int hidden, int vocab,
                                                         const __nv_bfloat16* __restrict__ gain,
                                                         const __nv_bfloat16* __restrict__ pos_table, int pos_offset,
                                                         float* __restrict__ part1) {
  griddep_wait();
  griddep_launch();
  const int t = blockIdx.x;
  const int id = ids[t];
  const bool pad = (pos != nullptr && pos[t] < 0) || id < 0 || id >= vocab;
  const __nv_bfloat16* row = table + (size_t)(pad ? 0 : id) * hidden;
  // OPT: learned absolute positions (row p + offset); part1: the row's sum (fused LayerNorm consumers)
  const __nv_bfloat16* prow = (pos_table && !pad) ? pos_table + (size_t)(pos[t] + pos_offset) * hidden : nullptr;
  float ss = 0.f, s1 = 0.f;
  if ((hidden & 7) == 0) {
    // 8 elements per thread: one 16-byte load per source row, 16-byte stores (one round trip)
    for (int i = threadIdx.x * 8; i < hidden; i += blockDim.x * 8) {
      float v[8];
      const uint4 r4 = pad ? make_uint4(0u, 0u, 0u, 0u) : *reinterpret_cast<const uint4*>(row + i);
      const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&r4);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = __bfloat162float(rb[e]);
      if (prow) {
        const uint4 p4 = *reinterpret_cast<const uint4*>(prow + i);
        const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&p4);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] += __bfloat162float(pb[e]);
      }
      float g[8] = {1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f};
      if (gain) {
        const uint4 g4 = *reinterpret_cast<const uint4*>(gain + i);
        const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&g4);
#pragma unroll
        for (int e = 0; e < 8; ++e) g[e] = __bfloat162float(gb[e]);
      }
      float4* hd = reinterpret_cast<float4*>(h + (size_t)t * hidden + i);
      hd[0] = make_float4(v[0], v[1], v[2], v[3]);
      hd[1] = make_float4(v[4], v[5], v[6], v[7]);
      uint4 o;
      __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        ob[e] = __float2bfloat16_rn(gain ? v[e] * g[e] : v[e]);
        ss += v[e] * v[e];
        s1 += v[e];
      }
      *reinterpret_cast<uint4*>(xb + (size_t)t * hidden + i) = o;
    }
  } else {
    for (int i = threadIdx.x; i < hidden; i += blockDim.x) {
      float v = pad ? 0.f : __bfloat162float(row[i]);
      if (prow) v += __bfloat162float(prow[i]);
      h[(size_t)t * hidden + i] = v;
      xb[(size_t)t * hidden + i] = __float2bfloat16_rn(gain ? v * __bfloat162float(gain[i]) : v);
      ss += v * v;
      s1 += v;
    }
  }
  __shared__ float red[8], red1[8];
  ss = warp_sum(ss);
  s1 = warp_sum(s1);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = ss;
    red1[threadIdx.x >> 5] = s1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f, tot1 = 0.f;
    for (int w = 0; w < 8; ++w) {
      tot += red[w];
      tot1 += red1[w];
    }
    part[t] = tot;
    if (part1) part1[t] = tot1;
  }
}

int launch_embed_norm(const void* table, const int32_t* ids, const int32_t* pos, float* h, void* xb, float* part,
                      int n_tok, int hidden, int vocab, cudaStream_t st, const void* gain, const void* pos_table,
                      int pos_offset, float* part1) {
  if (n_tok <= 0) return 0;
  if (pos_table && !pos) return SB_EINVAL;
  return launch_k(embed_norm_kernel, dim3(n_tok), dim3(256), 0, st, (const __nv_bfloat16*)table, ids, pos, h,
                  (__nv_bfloat16*)xb, part, hidden, vocab, (const __nv_bfloat16*)gain,
                  (const __nv_bfloat16*)pos_table, pos_offset, part1);
}

// ---------------------------------------------------------------- RMSNorm
// y[r] = dtype(x[src_row(r)] * rsqrt(mean(x^2) + eps) * g); src_row(r) = r*row_step + row_off.
// One CTA per row, the row held in registers as float4 (hidden <= 8192).
template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x, const T* __restrict__ g,
                                                      T* __restrict__ y, int hidden, float eps, int row_step,
                                                      int row_off) {
  griddep_wait();
  griddep_launch();
  const int r = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)(r * row_step + row_off) * hidden);
  const int n4 = hidden >> 2;
  float4 v[8];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    int i = threadIdx.x + c * 256;
    if (i < n4) {
      v[c] = xr[i];
      ss += v[c].x * v[c].x + v[c].y * v[c].y + v[c].z * v[c].z + v[c].w * v[c].w;
    }
  }
  __shared__ float red[8];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float inv = rsqrtf(tot / (float)hidden + eps);
  T* yr = y + (size_t)r * hidden;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    int i = threadIdx.x + c * 256;
    if (i < n4) {
      int e = i * 4;
      yr[e + 0] = from_f32<T>(v[c].x * inv * to_f32(g[e + 0]));
      yr[e + 1] = from_f32<T>(v[c].y * inv * to_f32(g[e + 1]));
      yr[e + 2] = from_f32<T>(v[c].z * inv * to_f32(g[e + 2]));
      yr[e + 3] = from_f32<T>(v[c].w * inv * to_f32(g[e + 3]));
    }
  }
}

int launch_rmsnorm(int dtype, const float* x, const void* g, void* y, int rows, int hidden, float eps, int row_step,
                   int row_off, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (hidden % 4 || hidden > 8192) return SB_EUNSUPPORTED;
  if (dtype == SB_BF16)
    return launch_k(rmsnorm_kernel<__nv_bfloat16>, dim3(rows), dim3(256), 0, st, x, (const __nv_bfloat16*)g,
                    (__nv_bfloat16*)y, hidden, eps, row_step, row_off);
  return launch_k(rmsnorm_kernel<float>, dim3(rows), dim3(256), 0, st, x, (const float*)g, (float*)y, hidden, eps,
                  row_step, row_off);
}

// ---------------------------------------------------------------- LayerNorm (OPT)
// y[r] = dtype((x - mean) * rsqrt(var + eps) * g + b), two passes over the row
// held in registers (float4, hidden <= 8192); src_row(r) = r*row_step + row_off.
template <typename T>
__global__ void __launch_bounds__(256) layernorm_kernel(const float* __restrict__ x, const T* __restrict__ g,
                                                        const T* __restrict__ b, T* __restrict__ y, int hidden,
                                                        float eps, int row_step, int row_off) {
  griddep_wait();
  griddep_launch();
  const int r = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)(r * row_step + row_off) * hidden);
  const int n4 = hidden >> 2;
  float4 v[8];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    int i = threadIdx.x + c * 256;
    if (i < n4) {
      v[c] = xr[i];
      s += (v[c].x + v[c].y) + (v[c].z + v[c].w);
    }
  }
  __shared__ float red[8];
  __shared__ float stat[2];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    stat[0] = t / (float)hidden;
  }
  __syncthreads();
  const float mean = stat[0];
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    int i = threadIdx.x + c * 256;
    if (i < n4) {
      const float a = v[c].x - mean, bb = v[c].y - mean, cc = v[c].z - mean, d = v[c].w - mean;
      q += (a * a + bb * bb) + (cc * cc + d * d);
    }
  }
  q = warp_sum(q);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    stat[1] = rsqrtf(t / (float)hidden + eps);
  }
  __syncthreads();
  const float inv = stat[1];
  T* yr = y + (size_t)r * hidden;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    int i = threadIdx.x + c * 256;
    if (i < n4) {
      int e = i * 4;
      yr[e + 0] = from_f32<T>((v[c].x - mean) * inv * to_f32(g[e + 0]) + to_f32(b[e + 0]));
      yr[e + 1] = from_f32<T>((v[c].y - mean) * inv * to_f32(g[e + 1]) + to_f32(b[e + 1]));
      yr[e + 2] = from_f32<T>((v[c].z - mean) * inv * to_f32(g[e + 2]) + to_f32(b[e + 2]));
      yr[e + 3] = from_f32<T>((v[c].w - mean) * inv * to_f32(g[e + 3]) + to_f32(b[e + 3]));
    }
  }
}

int launch_layernorm(int dtype, const float* x, const void* g, const void* b, void* y, int rows, int hidden, float eps,
                     int row_step, int row_off, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (hidden % 4 || hidden > 8192 || !g || !b) return SB_EUNSUPPORTED;
  if (dtype == SB_BF16)
    return launch_k(layernorm_kernel<__nv_bfloat16>, dim3(rows), dim3(256), 0, st, x, (const __nv_bfloat16*)g,
                    (const __nv_bfloat16*)b, (__nv_bfloat16*)y, hidden, eps, row_step, row_off);
  return launch_k(layernorm_kernel<float>, dim3(rows), dim3(256), 0, st, x, (const float*)g, (const float*)b,
                  (float*)y, hidden, eps, row_step, row_off);
}

// ---------------------------------------------------------------- RoPE + KV append
// qkv [T, (nq + 2 nkv) * hd] -> q_out [T, nq*hd] rotated; K rotated and V written
// to cache[layer][slot][kvh][pos][hd].  rotate-half convention (HF Llama):
//   out[i]      = x[i] cos - x[i+hd/2] sin
//   out[i+hd/2] = x[i+hd/2] cos + x[i] sin
template <typename T>
__global__ void rope_append_kernel(const T* __restrict__ qkv, T* __restrict__ q_out, T* __restrict__ kc,
                                   T* __restrict__ vc, const int32_t* __restrict__ tok_slot,
                                   const int32_t* __restrict__ tok_pos, const float* __restrict__ cosT,
                                   const float* __restrict__ sinT, int q_len, int nq, int nkv, int hd,
                                   int ctx_max, int max_pos) {
  griddep_wait();
  griddep_launch();
  int t = blockIdx.x;
  int slot = tok_slot[t / q_len];
  int p = tok_pos[t];
  int half = hd / 2;
  const T* row = qkv + (size_t)t * (nq + 2 * nkv) * hd;
  int pc = p < 0 ? 0 : (p >= max_pos ? max_pos - 1 : p);
  const float* cr = cosT + (size_t)pc * half;
  const float* sr = sinT + (size_t)pc * half;
  for (int e = threadIdx.x; e < nq * half; e += blockDim.x) {
    int h = e / half, i = e % half;
    const T* src = row + h * hd;
    float a = to_f32(src[i]), b = to_f32(src[i + half]);
    float c = cr[i], s = sr[i];
    T* dst = q_out + (size_t)t * nq * hd + h * hd;
    dst[i] = from_f32<T>(a * c - b * s);
    dst[i + half] = from_f32<T>(b * c + a * s);
  }
  if (p < 0) return;  // padding token: nothing enters the cache
  for (int e = threadIdx.x; e < nkv * half; e += blockDim.x) {
    int h = e / half, i = e % half;
    const T* src = row + (nq + h) * hd;
    float a = to_f32(src[i]), b = to_f32(src[i + half]);
    float c = cr[i], s = sr[i];
    T* dst = kc + (((size_t)slot * nkv + h) * ctx_max + p) * hd;
    dst[i] = from_f32<T>(a * c - b * s);
    dst[i + half] = from_f32<T>(b * c + a * s);
  }
  for (int e = threadIdx.x; e < nkv * hd; e += blockDim.x) {
    int h = e / hd, i = e % hd;
    vc[(((size_t)slot * nkv + h) * ctx_max + p) * hd + i] = row[(nq + nkv + h) * hd + i];
  }
}

// bf16, 16-byte vectors: a thread rotates 8 (x_i, x_{i+hd/2}) pairs of one head
// (two 16-byte loads + 2 x 2 float4 of cos / sin) -- same arithmetic as above.
__global__ void __launch_bounds__(256) rope_append_vec_kernel(
    const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ kc,
    __nv_bfloat16* __restrict__ vc, const int32_t* __restrict__ tok_slot, const int32_t* __restrict__ tok_pos,
    const float* __restrict__ cosT, const float* __restrict__ sinT, int q_len, int nq, int nkv, int hd, int ctx_max,
    int max_pos) {
  griddep_wait();
  griddep_launch();
  const int t = blockIdx.x;
  const int slot = tok_slot[t / q_len];
  const int p = tok_pos[t];
  const int half = hd / 2, cpr = half / 8;
  const __nv_bfloat16* row = qkv + (size_t)t * (nq + 2 * nkv) * hd;
  const int pc = p < 0 ? 0 : (p >= max_pos ? max_pos - 1 : p);
  const float* cr = cosT + (size_t)pc * half;
  const float* sr = sinT + (size_t)pc * half;
  const int n_rot = (p < 0 ? nq : nq + nkv) * cpr;  // padding token: nothing enters the cache
  for (int e = threadIdx.x; e < n_rot; e += blockDim.x) {
    const int h = e / cpr, c8 = (e % cpr) * 8;
    const __nv_bfloat16* src = row + h * hd + c8;
    const uint4 u0 = *reinterpret_cast<const uint4*>(src), u1 = *reinterpret_cast<const uint4*>(src + half);
    const float4 c0 = *reinterpret_cast<const float4*>(cr + c8), c1 = *reinterpret_cast<const float4*>(cr + c8 + 4);
    const float4 s0 = *reinterpret_cast<const float4*>(sr + c8), s1 = *reinterpret_cast<const float4*>(sr + c8 + 4);
    const __nv_bfloat16* x0 = reinterpret_cast<const __nv_bfloat16*>(&u0);
    const __nv_bfloat16* x1 = reinterpret_cast<const __nv_bfloat16*>(&u1);
    const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const float ss[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    uint4 oa, ob;
    __nv_bfloat16* pa = reinterpret_cast<__nv_bfloat16*>(&oa);
    __nv_bfloat16* pb = reinterpret_cast<__nv_bfloat16*>(&ob);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float a = __bfloat162float(x0[i]), b = __bfloat162float(x1[i]);
      pa[i] = __float2bfloat16_rn(a * cc[i] - b * ss[i]);
      pb[i] = __float2bfloat16_rn(b * cc[i] + a * ss[i]);
    }
    __nv_bfloat16* dst = h < nq ? q_out + ((size_t)t * nq + h) * hd
                                : kc + (((size_t)slot * nkv + (h - nq)) * ctx_max + p) * hd;
    *reinterpret_cast<uint4*>(dst + c8) = oa;
    *reinterpret_cast<uint4*>(dst + half + c8) = ob;
  }
  if (p < 0) return;
  const int vpr = hd / 8;
  for (int e = threadIdx.x; e < nkv * vpr; e += blockDim.x) {
    const int h = e / vpr, c = (e % vpr) * 8;
    *reinterpret_cast<uint4*>(vc + (((size_t)slot * nkv + h) * ctx_max + p) * hd + c) =
        *reinterpret_cast<const uint4*>(row + (nq + nkv + h) * hd + c);
  }
}

int launch_rope_append(int dtype, const void* qkv, void* q_out, void* kc, void* vc, const int32_t* tok_slot,
                       const int32_t* tok_pos, const float* cosT, const float* sinT, int n_tok, int q_len, int nq,
                       int nkv, int hd, int ctx_max, int max_pos, cudaStream_t st) {
  if (n_tok <= 0) return 0;
  if (dtype == SB_BF16 && hd % 16 == 0)
    return launch_k(rope_append_vec_kernel, dim3(n_tok), dim3(128), 0, st, (const __nv_bfloat16*)qkv,
                    (__nv_bfloat16*)q_out, (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, tok_slot, tok_pos, cosT, sinT,
                    q_len, nq, nkv, hd, ctx_max, max_pos);
  if (dtype == SB_BF16)
    return launch_k(rope_append_kernel<__nv_bfloat16>, dim3(n_tok), dim3(256), 0, st, (const __nv_bfloat16*)qkv,
                    (__nv_bfloat16*)q_out, (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, tok_slot, tok_pos, cosT, sinT,
                    q_len, nq, nkv, hd, ctx_max, max_pos);
  return launch_k(rope_append_kernel<float>, dim3(n_tok), dim3(256), 0, st, (const float*)qkv, (float*)q_out,
                  (float*)kc, (float*)vc, tok_slot, tok_pos, cosT, sinT, q_len, nq, nkv, hd, ctx_max, max_pos);
}

// ---------------------------------------------------------------- attention (K3)
// One CTA per (q head, sequence, group of QG queries); 128 threads.  Keys of
// the slot stream through shared memory in 64-key tiles (16-byte vector loads;
// row stride padded to 136 elements so 16-byte smem reads are conflict-free).
// Query j at absolute position p_j sees keys [0, p_j]: the causal mask inside
// the speculative window.  Online softmax in fp32 with a fixed key order
// (64-key tiles, ascending) -> a query's output is independent of how many
// other queries share the launch (batch invariance, spec == greedy in fp32).
constexpr int kAttnKT = 64;

template <typename T> struct AttnVec;  // elements per 16-byte vector
template <> struct AttnVec<__nv_bfloat16> { static constexpr int n = 8; };
template <> struct AttnVec<float> { static constexpr int n = 4; };

template <typename T, int HD, int QG>
__global__ void __launch_bounds__(128) attention_kernel(const T* __restrict__ q, const T* __restrict__ kc,
                                                        const T* __restrict__ vc, T* __restrict__ out,
                                                        const int32_t* __restrict__ tok_slot,
                                                        const int32_t* __restrict__ tok_pos, int q_len, int nq,
                                                        int nkv, int ctx_max, float scale) {
  constexpr int VE = AttnVec<T>::n;           // elements per 16B
  constexpr int KS = HD + 16 / (int)sizeof(T) * 1;  // padded row stride (elements): +16 bytes
  // dynamic shared memory (fp32 at head_dim 128 needs ~78 KB): K tile | V tile | Q | S
  extern __shared__ __align__(16) unsigned char attn_smem[];
  T(*Ks)[KS] = reinterpret_cast<T(*)[KS]>(attn_smem);
  T(*Vs)[HD] = reinterpret_cast<T(*)[HD]>(attn_smem + sizeof(T) * kAttnKT * KS);
  float(*Qs)[HD] = reinterpret_cast<float(*)[HD]>(attn_smem + sizeof(T) * kAttnKT * (KS + HD));
  float(*S)[kAttnKT] = reinterpret_cast<float(*)[kAttnKT]>(attn_smem + sizeof(T) * kAttnKT * (KS + HD) +
                                                           sizeof(float) * QG * HD);
  __shared__ float m_run[QG], l_run[QG], corr[QG];
  __shared__ int qpos[QG];
  griddep_wait();
  griddep_launch();

  const int head = blockIdx.x, seq = blockIdx.y, qg = blockIdx.z;
  const int kvh = head / (nq / nkv);
  const int slot = tok_slot[seq];
  const int tid = threadIdx.x;
  const int j0 = qg * QG;
  const int nqg = min(QG, q_len - j0);
  if (nqg <= 0) return;

  if (tid < QG) {
    qpos[tid] = tid < nqg ? tok_pos[seq * q_len + j0 + tid] : -1;
    m_run[tid] = -INFINITY;
    l_run[tid] = 0.f;
  }
  for (int e = tid; e < QG * HD; e += 128) {
    int j = e / HD, d = e % HD;
    float v = 0.f;
    if (j < nqg) v = to_f32(q[((size_t)(seq * q_len + j0 + j) * nq + head) * HD + d]) * scale;
    Qs[j][d] = v;
  }
  __syncthreads();
  int maxp = -1;
#pragma unroll
  for (int j = 0; j < QG; ++j) maxp = max(maxp, qpos[j]);

  constexpr int DPT = (HD + 127) / 128;  // output dims per thread
  float acc[QG][DPT];
#pragma unroll
  for (int j = 0; j < QG; ++j)
#pragma unroll
    for (int c = 0; c < DPT; ++c) acc[j][c] = 0.f;

  const T* kbase = kc + ((size_t)slot * nkv + kvh) * ctx_max * HD;
  const T* vbase = vc + ((size_t)slot * nkv + kvh) * ctx_max * HD;
  const int n_keys = maxp + 1;
  constexpr int VPR = HD / VE;  // vectors per row

  for (int k0 = 0; k0 < n_keys; k0 += kAttnKT) {
    const int nk = min(kAttnKT, n_keys - k0);
    for (int e = tid; e < kAttnKT * VPR; e += 128) {
      int r = e / VPR, c = (e % VPR) * VE;
      uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
      if (r < nk) {
        kv = *reinterpret_cast<const uint4*>(kbase + (size_t)(k0 + r) * HD + c);
        vv = *reinterpret_cast<const uint4*>(vbase + (size_t)(k0 + r) * HD + c);
      }
      *reinterpret_cast<uint4*>(&Ks[r][c]) = kv;
      *reinterpret_cast<uint4*>(&Vs[r][c]) = vv;
    }
    __syncthreads();
    // scores: thread -> key r = tid % 64, queries j = tid/64 + 2i
    {
      const int r = tid & (kAttnKT - 1);
      const int jb = tid >> 6;
      float sc[QG];
#pragma unroll
      for (int j = 0; j < QG; ++j) sc[j] = 0.f;
#pragma unroll 4
      for (int c = 0; c < HD; c += VE) {
        uint4 raw = *reinterpret_cast<const uint4*>(&Ks[r][c]);
        const T* kv = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          float kf = to_f32(kv[e]);
#pragma unroll
          for (int j = 0; j < QG; ++j)
            if ((j & 1) == jb) sc[j] = fmaf(Qs[j][c + e], kf, sc[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < QG; ++j)
        if ((j & 1) == jb) S[j][r] = (r < nk && k0 + r <= qpos[j]) ? sc[j] : -INFINITY;
    }
    __syncthreads();
    // online softmax: warp w handles queries w, w+4, ...
    {
      const int w = tid >> 5, lane = tid & 31;
      for (int j = w; j < QG; j += 4) {
        float a = S[j][lane], b = S[j][lane + 32];
        float mt = warp_max(fmaxf(a, b));
        float mo = m_run[j];
        float mn = fmaxf(mo, mt);
        float ea = (mn == -INFINITY) ? 0.f : __expf(a - mn);
        float eb = (mn == -INFINITY) ? 0.f : __expf(b - mn);
        S[j][lane] = ea;
        S[j][lane + 32] = eb;
        float sum = warp_sum(ea + eb);
        if (lane == 0) {
          float cf = (mo == -INFINITY) ? 0.f : __expf(mo - mn);
          corr[j] = cf;
          l_run[j] = l_run[j] * cf + sum;
          m_run[j] = mn;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < QG; ++j)
#pragma unroll
      for (int c = 0; c < DPT; ++c) acc[j][c] *= corr[j];
    for (int r = 0; r < nk; ++r) {
#pragma unroll
      for (int c = 0; c < DPT; ++c) {
        int d = tid + c * 128;
        if (d < HD) {
          float vv = to_f32(Vs[r][d]);
#pragma unroll
          for (int j = 0; j < QG; ++j) acc[j][c] = fmaf(S[j][r], vv, acc[j][c]);
        }
      }
    }
    __syncthreads();
  }
  for (int j = 0; j < nqg; ++j) {
    float l = l_run[j];
#pragma unroll
    for (int c = 0; c < DPT; ++c) {
      int d = tid + c * 128;
      if (d < HD) out[((size_t)(seq * q_len + j0 + j) * nq + head) * HD + d] = from_f32<T>(l > 0.f ? acc[j][c] / l : 0.f);
    }
  }
}

// dynamic shared memory of attention_kernel<T, HD, QG> (opted in by attention_tc_init)
template <typename T, int HD, int QG>
constexpr size_t attn_simt_smem() {
  return sizeof(T) * kAttnKT * (2 * HD + 16 / sizeof(T)) + sizeof(float) * QG * (HD + kAttnKT);
}

template <typename T, int HD>
static cudaError_t attn_simt_attr() {
  cudaError_t e = cudaSuccess;
#define SB_ATTN_SIMT_ATTR(QG)                                                                                   \
  if (e == cudaSuccess)                                                                                         \
  e = cudaFuncSetAttribute(attention_kernel<T, HD, QG>, cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                           (int)attn_simt_smem<T, HD, QG>())
  SB_ATTN_SIMT_ATTR(1);
  SB_ATTN_SIMT_ATTR(2);
  SB_ATTN_SIMT_ATTR(4);
  SB_ATTN_SIMT_ATTR(8);
  SB_ATTN_SIMT_ATTR(16);
#undef SB_ATTN_SIMT_ATTR
  return e;
}

template <typename T, int HD>
static int attn_dispatch(int q_len, dim3 grid_xy, const void* q, const void* kc, const void* vc, void* out,
                         const int32_t* slot, const int32_t* pos, int nq, int nkv, int ctx, float scale,
                         cudaStream_t st) {
#define SB_ATTN(QG)                                                                                          \
  return launch_k(attention_kernel<T, HD, QG>, dim3(grid_xy.x, grid_xy.y, (q_len + QG - 1) / QG), dim3(128),   \
                  attn_simt_smem<T, HD, QG>(), st, (const T*)q, (const T*)kc, (const T*)vc, (T*)out, slot, pos,   \
                  q_len, nq, nkv, ctx, scale)
  if (q_len <= 1) SB_ATTN(1);
  if (q_len <= 2) SB_ATTN(2);
  if (q_len <= 4) SB_ATTN(4);
  if (q_len <= 8) SB_ATTN(8);
  SB_ATTN(16);
#undef SB_ATTN
}

int launch_attention(int dtype, const void* q, const void* kc, const void* vc, void* out, const int32_t* tok_slot,
                     const int32_t* tok_pos, int n_seq, int q_len, int nq, int nkv, int hd, int ctx_max,
                     cudaStream_t st) {
  if ((hd != 64 && hd != 128) || nq % nkv != 0) return SB_EUNSUPPORTED;
  dim3 g(nq, n_seq, 1);
  float scale = 1.0f / sqrtf((float)hd);
  if (dtype == SB_BF16)
    return hd == 128 ? attn_dispatch<__nv_bfloat16, 128>(q_len, g, q, kc, vc, out, tok_slot, tok_pos, nq, nkv, ctx_max,
                                                         scale, st)
                     : attn_dispatch<__nv_bfloat16, 64>(q_len, g, q, kc, vc, out, tok_slot, tok_pos, nq, nkv, ctx_max,
                                                        scale, st);
  return hd == 128 ? attn_dispatch<float, 128>(q_len, g, q, kc, vc, out, tok_slot, tok_pos, nq, nkv, ctx_max, scale, st)
                   : attn_dispatch<float, 64>(q_len, g, q, kc, vc, out, tok_slot, tok_pos, nq, nkv, ctx_max, scale, st);
}

// ---------------------------------------------------------------- tensor-core flash decoding (bf16)
// CTA = (kv head, sequence): all q heads of the kv group x all window tokens
// (<= 16 queries) form ONE 16-row MMA tile.  4 warps; warp w owns keys
// [16w, 16w+16) of every 64-key tile (split over keys, combined at the end in
// warp order -> deterministic).  S = Q K^T and O += P V with
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate; P is fed from the S
// accumulators without a smem round trip).  KV tiles stream through a 3-stage
// cp.async ring; padded 272-byte rows make every ldmatrix conflict-free.  The
// prologue rotates Q (RoPE, rounded to bf16) and appends this forward's
// rotated K / V rows to the cache (this CTA is the only reader of its slab).
constexpr int kTcStages = 3;
int g_attn_splits = 1;  // 1 off (default: measured +10% slower at b=1..8), 0 auto, n forced (sb_set_attention_splits)
// KV loads of a model whose weights stream evict-first (the target) are evict-first too
// (env SB_ATTN_KV_L2HINT=0/1 overrides)
static int g_kv_l2_hint() {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("SB_ATTN_KV_L2HINT");
    env = e ? atoi(e) : -1;
  }
  return env >= 0 ? env : (g_w_l2_hint == 1 ? 1 : 0);
}
int g_attn_l2pf = -1;   // -1: from env SB_ATTN_L2PF (default off)

int g_attn_stages = -1;  // ring stages (3, 4 or 6) when the grid fits one CTA per SM: -1 env SB_ATTN_STAGES

// BLK: prefill blocks (A.qr set); SPLIT: flash-decoding key splits (gridDim.z > 1) -- compile-time, so
// each launch carries only its own paths (one inlined item; the instruction cache holds it).
template <int HD, int STAGES, bool BLK, bool SPLIT>
__global__ void __launch_bounds__(128) attention_tc_kernel(AttnArgs A) {
  extern __shared__ __align__(128) uint8_t tsm[];
  __shared__ AttnShared sh;
  __shared__ unsigned long long tr_t[4];
  if (A.trace && threadIdx.x == 0) tr_t[0] = tr_t[2] = tr_t[3] = gtime();
  if (A.l2_next && threadIdx.x < 32) {
    // The attention reads little (KV history) and waits a lot: keep HBM busy by
    // pulling this CTA's share of the next GEMM's weights into L2 (bulk prefetch,
    // no smem, no completion to wait for).  Weights are constant: legal before
    // the PDL wait.
    const unsigned long long nblk = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
    const unsigned long long b = blockIdx.x + gridDim.x * (blockIdx.y + (unsigned long long)gridDim.y * blockIdx.z);
    const unsigned long long per = ((A.l2_next_bytes + nblk - 1) / nblk + 4095) & ~4095ull;
    const unsigned long long lo = b * per, hi = min(lo + per, A.l2_next_bytes);
    for (unsigned long long o = lo + threadIdx.x * 16384ull; o < hi; o += 32 * 16384ull) {
      const unsigned n = (unsigned)min(16384ull, hi - o);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.l2_next + o), "r"(n) : "memory");
    }
  }
  AttnArgs B = A;
  B.tr_t = tr_t;
  if (BLK)
    attn_tc_item<HD, STAGES, true, false>(B, blockIdx.x, blockIdx.y, 0, 1, tsm, sh, threadIdx.x, true, blockIdx.z);
  else
    attn_tc_item<HD, STAGES, false, SPLIT>(B, blockIdx.x, blockIdx.y, SPLIT ? (int)blockIdx.z : 0,
                                           SPLIT ? (int)gridDim.z : 1, tsm, sh, threadIdx.x, true);
  if (A.trace) {
    __syncthreads();
    if (threadIdx.x == 0) cta_trace_write(A.trace, A.trace_id, 2, tr_t);
  }
}

// A decode grid of at most one CTA per SM reserves this much shared memory per CTA, so that no two of its
// CTAs share an SM (launched early under PDL, beside the qkv GEMM's CTAs, they were otherwise packed three
// to an SM: 96 CTAs on 32 SMs for the draft step).
constexpr size_t kAttnSpreadBytes = 120 * 1024;
static int g_attn_spread = -1;
// Opt every ring variant in to its dynamic shared memory once (outside graph capture).
int attention_tc_init() {
  static int rc = -1;
  if (rc < 0) {
    cudaError_t e = cudaSuccess;
#define SB_ATTN_ATTR(H, S)                                                                                        \
  if (e == cudaSuccess)                                                                                           \
    e = cudaFuncSetAttribute(attention_tc_kernel<H, S, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)(TcAttnSmem<H, S>::bytes > kAttnSpreadBytes ? TcAttnSmem<H, S>::bytes : kAttnSpreadBytes)); \
  if (e == cudaSuccess)                                                                                           \
    e = cudaFuncSetAttribute(attention_tc_kernel<H, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                             (int)TcAttnSmem<H, S>::bytes);                                                        \
  if (e == cudaSuccess)                                                                                           \
    e = cudaFuncSetAttribute(attention_tc_kernel<H, S, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                             (int)TcAttnSmem<H, S>::bytes)
    SB_ATTN_ATTR(128, 2);
    SB_ATTN_ATTR(128, 3);
    SB_ATTN_ATTR(128, 4);
    SB_ATTN_ATTR(64, 2);
    SB_ATTN_ATTR(64, 3);
    SB_ATTN_ATTR(64, 4);
    if (e == cudaSuccess) e = attn_simt_attr<__nv_bfloat16, 64>();
    if (e == cudaSuccess) e = attn_simt_attr<__nv_bfloat16, 128>();
    if (e == cudaSuccess) e = attn_simt_attr<float, 64>();
    if (e == cudaSuccess) e = attn_simt_attr<float, 128>();
#undef SB_ATTN_ATTR
    rc = e == cudaSuccess ? 0 : (int)e;
  }
  return rc;
}

// Launch attention_tc_kernel over grid (nkv, n_seq, z) with the ring depth for its residency.
static int launch_attn_grid(const AttnArgs& A0, int hd, int n_seq, int z, cudaStream_t st) {
  AttnArgs A = A0;
  A.trace = g_cta_trace;
  A.trace_id = g_cta_trace ? g_cta_trace_seq++ : 0;
  A.tr_t = nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(A.nkv, n_seq, z);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  if (g_attn_stages < 0) {
    const char* e = getenv("SB_ATTN_STAGES");
    g_attn_stages = e ? atoi(e) : 4;  // measured: 4 and 6 tie, 3-5% over 3 at b = 2..4
  }
  const int ctas = A.nkv * n_seq * z;
  static int multi = -1;  // ring depth beyond two CTAs per SM (env SB_ATTN_STAGES_MULTI)
  if (multi < 0) {
    const char* e = getenv("SB_ATTN_STAGES_MULTI");
    multi = e ? atoi(e) : 2;
  }
  // deepest ring that keeps the grid in one wave: 4 stages at <= 1 CTA per SM, 3 (2 per SM), then 2
  // (3 per SM; measured: b=64,k=2 verify 6.72 -> 6.23 ms, b=32,k=2 4.61 -> 4.40 ms)
  const int stages = ctas <= num_sms() ? g_attn_stages : ctas <= 2 * num_sms() ? 3 : multi;
  {  // normally done by gemm_tc_init outside capture; relaxed so a first call inside a capture is legal
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    const int rc = attention_tc_init();
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (rc) return rc;
  }
  if (g_attn_spread < 0) {
    const char* e = getenv("SB_ATTN_SPREAD");
    g_attn_spread = e ? atoi(e) : 1;
  }
  const bool spread = g_attn_spread && ctas <= num_sms() && A.qr == nullptr && z == 1;
  auto go = [&](void (*kern)(AttnArgs), size_t bytes) {
    cfg.dynamicSmemBytes = spread && bytes < kAttnSpreadBytes ? kAttnSpreadBytes : bytes;
    return cudaLaunchKernelEx(&cfg, kern, A);
  };
  const bool blk = A.qr != nullptr, spl = z > 1 && !blk;
#define SB_ATTN_GO(H, S) \
  (blk ? go(attention_tc_kernel<H, S, true, false>, TcAttnSmem<H, S>::bytes) \
       : spl ? go(attention_tc_kernel<H, S, false, true>, TcAttnSmem<H, S>::bytes) \
             : go(attention_tc_kernel<H, S, false, false>, TcAttnSmem<H, S>::bytes))
  cudaError_t e;
  if (hd == 128) e = stages >= 4 ? SB_ATTN_GO(128, 4) : stages == 3 ? SB_ATTN_GO(128, 3) : SB_ATTN_GO(128, 2);
  else e = stages >= 4 ? SB_ATTN_GO(64, 4) : stages == 3 ? SB_ATTN_GO(64, 3) : SB_ATTN_GO(64, 2);
#undef SB_ATTN_GO
  if (e != cudaSuccess) return (int)e;
  ++g_kernel_count;
  return 0;
}

int launch_attention_tc(const void* qkv, void* kc, void* vc, void* out, const int32_t* tok_slot, const int32_t* tok_pos,
                        const float* cosT, const float* sinT, int n_seq, int q_len, int nq, int nkv, int hd,
                        int ctx_max, int max_pos, cudaStream_t st, const AttnScratch* scratch,
                        const void* l2_next, size_t l2_next_bytes) {
  if (g_attn_l2pf < 0) {
    const char* e = getenv("SB_ATTN_L2PF");
    g_attn_l2pf = e ? atoi(e) : 0;  // measured: no gain at b=8, -5% at b=1 (opt-in)
  }
  if (!g_attn_l2pf || (l2_next_bytes & 15)) l2_next = nullptr;
  if ((hd != 64 && hd != 128) || nq % nkv != 0 || (nq / nkv) * q_len > 16) return SB_EUNSUPPORTED;
  const float scale = 1.0f / sqrtf((float)hd);
  // key splits: enough CTAs for ~2 per SM, at most what the scratch holds, and
  // at least 2 key tiles of the full context per split
  int splits = 1;
  if (scratch && scratch->part && g_attn_splits != 1) {
    const int items = n_seq * nkv;
    splits = g_attn_splits > 1 ? g_attn_splits : (2 * 148 + items - 1) / items;
    const int max_tiles = (ctx_max + kTcKT - 1) / kTcKT;
    if (splits > max_tiles / 2) splits = max_tiles / 2;
    if (splits > 8) splits = 8;
    while (splits > 1 && items * splits > scratch->max_entries) --splits;
    if (items > scratch->max_items) splits = 1;
    if (splits < 1) splits = 1;
  }
  AttnSplit sp{scratch ? scratch->part : nullptr, scratch ? scratch->ml : nullptr,
               scratch ? scratch->counter : nullptr};
  AttnArgs A{(const __nv_bfloat16*)qkv, (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, (__nv_bfloat16*)out, tok_slot, tok_pos,
             cosT, sinT, q_len, nq, nkv, ctx_max, max_pos, scale, sp, (const char*)l2_next,
             l2_next ? (unsigned long long)l2_next_bytes : 0ull, nullptr, 0, g_kv_l2_hint()};
  return launch_attn_grid(A, hd, n_seq, splits, st);
}

// Prefill-sized windows (after launch_rope_append): tensor-core flash attention
// over blocks of 16 / group query tokens per CTA, causal by position.
int launch_attention_tc_prefill(const void* qr, void* kc, void* vc, void* out, const int32_t* tok_slot,
                                const int32_t* tok_pos, int n_seq, int q_len, int nq, int nkv, int hd, int ctx_max,
                                cudaStream_t st) {
  if ((hd != 64 && hd != 128) || nq % nkv != 0 || nq / nkv > 16 || q_len < 1) return SB_EUNSUPPORTED;
  const int q_blk = 16 / (nq / nkv);
  const int nblk = (q_len + q_blk - 1) / q_blk;
  if (nblk > 65535) return SB_EUNSUPPORTED;
  AttnArgs A{nullptr, (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, (__nv_bfloat16*)out, tok_slot, tok_pos, nullptr, nullptr,
             q_len, nq, nkv, ctx_max, 1, 1.0f / sqrtf((float)hd), AttnSplit{nullptr, nullptr, nullptr}, nullptr, 0ull,
             (const __nv_bfloat16*)qr, q_blk, 0};  // (the L2 hint faulted here on wide-GQA blocks: off)
  return launch_attn_grid(A, hd, n_seq, nblk, st);
}

// ---------------------------------------------------------------- KV compaction (K5)
// One (slab pair, layer) per blockIdx (y, z): copy positions [0, len) of every
// kv head of slot src -> slot dst, K and V, in 16-byte vectors (a position row
// is hd * elem_size = 128 / 256 / 512 bytes).  dst slots must not be sources of
// the same call (compaction moves live rows into freed slots).
__global__ void kv_compact_kernel(uint4* __restrict__ k, uint4* __restrict__ v, const int32_t* __restrict__ src,
                                  const int32_t* __restrict__ dst, const int32_t* __restrict__ len, int slots,
                                  int nkv, size_t slab_vec, size_t row_vec) {
  griddep_wait();
  griddep_launch();
  const int i = blockIdx.y, layer = blockIdx.z;
  const int s = src[i], d = dst[i];
  if (s == d) return;
  const size_t per = (size_t)len[i] * row_vec;
  for (int h = 0; h < nkv; ++h) {
    const size_t so = (((size_t)layer * slots + s) * nkv + h) * slab_vec;
    const size_t doff = (((size_t)layer * slots + d) * nkv + h) * slab_vec;
    for (size_t e = blockIdx.x * blockDim.x + threadIdx.x; e < per; e += (size_t)gridDim.x * blockDim.x) {
      k[doff + e] = k[so + e];
      v[doff + e] = v[so + e];
    }
  }
}

int launch_kv_compact(int dtype, void* k, void* v, const int32_t* src, const int32_t* dst, const int32_t* len, int n,
                      int layers, int slots, int nkv, int ctx_max, int hd, cudaStream_t st) {
  if (n <= 0) return 0;
  const size_t es = dtype == SB_BF16 ? 2 : 4;
  if ((hd * es) % 16) return SB_EUNSUPPORTED;
  const size_t row_vec = hd * es / 16;
  dim3 grid(8, n, layers);
  return launch_k(kv_compact_kernel, grid, dim3(256), 0, st, (uint4*)k, (uint4*)v, src, dst, len, slots, nkv,
                  (size_t)ctx_max * row_vec, row_vec);
}

}  // namespace sb

// ---------------------------------------------------------------- tensor-parallel glue
namespace sb {

// After the all-reduce of a row-parallel projection: resid += part; on the
// fused-norm path also the bf16 residual copy and the per-128-column
// sum-of-squares partials npart[tile][t] the next GEMM's 1/rms reads.
// grid (T, ceil(H/128)), 128 threads: one element per thread, fixed-order sums.
// part is the all-reduced update: fp32, or bf16 when part_bf16 (the bf16 model's exchange dtype).
__global__ void __launch_bounds__(128) tp_resid_add_kernel(float* __restrict__ resid, const void* __restrict__ part,
                                                           int part_bf16, __nv_bfloat16* __restrict__ xb,
                                                           float* __restrict__ npart, int T, int H,
                                                           const __nv_bfloat16* __restrict__ gain) {
  griddep_wait();
  griddep_launch();
  const int t = blockIdx.x, tile = blockIdx.y;
  const int col = tile * 128 + threadIdx.x;
  float nv = 0.f;
  if (col < H) {
    const size_t o = (size_t)t * H + col;
    const float pv = part_bf16 ? __bfloat162float(((const __nv_bfloat16*)part)[o]) : ((const float*)part)[o];
    nv = resid[o] + pv;
    resid[o] = nv;
    if (xb) xb[o] = __float2bfloat16_rn(gain ? nv * __bfloat162float(gain[col]) : nv);
  }
  if (!npart) return;
  __shared__ float red[4];
  const float s = warp_sum(nv * nv);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) npart[(size_t)tile * T + t] = ((red[0] + red[1]) + red[2]) + red[3];
}

int launch_tp_resid_add(float* resid, const void* part, int part_bf16, void* xb, float* npart, int T, int H,
                        cudaStream_t st, const void* gain) {
  if (T <= 0) return 0;
  return launch_k(tp_resid_add_kernel, dim3(T, (H + 127) / 128), dim3(128), 0, st, resid, part, part_bf16,
                  (__nv_bfloat16*)xb, npart, T, H, (const __nv_bfloat16*)gain);
}

// Vocab-parallel greedy lm_head.  pack: this rank's per-128-row argmax partials [n_tiles][rows]
// -> one (value, global index) pair per row, pair[r] = {v, bits(i + vocab_off)} (the all-gather
// payload: 8 bytes per row instead of the logits row).  final: merge the world gathered pairs
// [world][rows][2] (ties -> lowest global index: identical to an argmax of the full row).
// idx == NULL: val is this rank's raw logits slice [rows][n_tiles] (fp32 path: no fused partials) and
// the column is the local index.
__global__ void tp_argmax_pack_kernel(const float* __restrict__ val, const int* __restrict__ idx, int n_tiles, int rows,
                                      int vocab_off, float2* __restrict__ pair) {
  griddep_wait();
  griddep_launch();
  const int r = blockIdx.x, lane = threadIdx.x;
  ArgMax a{-INFINITY, INT_MAX};
  if (idx)
    for (int t = lane; t < n_tiles; t += 32) a = argmax_merge(a, ArgMax{val[(size_t)t * rows + r], idx[(size_t)t * rows + r]});
  else
    for (int t = lane; t < n_tiles; t += 32) a = argmax_merge(a, ArgMax{val[(size_t)r * n_tiles + t], t});
  a = warp_argmax(a);
  if (lane == 0) pair[r] = make_float2(a.v, __int_as_float(a.i == INT_MAX ? INT_MAX : a.i + vocab_off));
}

__global__ void tp_argmax_final_kernel(const float2* __restrict__ pairs, int world, int rows, int32_t* out_tok,
                                       int out_stride, int32_t* next_ids, int32_t* next_pos,
                                       const int32_t* base_pos, int pos_offset) {
  griddep_wait();
  griddep_launch();
  const int r = blockIdx.x, lane = threadIdx.x;
  ArgMax a{-INFINITY, INT_MAX};
  for (int w = lane; w < world; w += 32) {
    const float2 pr = pairs[(size_t)w * rows + r];
    a = argmax_merge(a, ArgMax{pr.x, __float_as_int(pr.y)});
  }
  a = warp_argmax(a);
  if (lane == 0) {
    if (out_tok) out_tok[(size_t)r * out_stride] = a.i;
    if (next_ids) next_ids[r] = a.i;
    if (next_pos) next_pos[r] = base_pos[r] + pos_offset;
  }
}

int launch_tp_argmax_pack(const float* val, const int* idx, int n_tiles, int rows, int vocab_off, float* pair,
                          cudaStream_t st) {
  if (rows <= 0) return 0;
  return launch_k(tp_argmax_pack_kernel, dim3(rows), dim3(32), 0, st, val, idx, n_tiles, rows, vocab_off,
                  (float2*)pair);
}

int launch_tp_argmax_final(const float* pairs, int world, int rows, int32_t* out_tok, int out_stride,
                           int32_t* next_ids, int32_t* next_pos, const int32_t* base_pos, int pos_offset,
                           cudaStream_t st) {
  if (rows <= 0) return 0;
  return launch_k(tp_argmax_final_kernel, dim3(rows), dim3(32), 0, st, (const float2*)pairs, world, rows, out_tok,
                  out_stride, next_ids, next_pos, base_pos, pos_offset);
}

// all_gather output [world][rows][Vl] -> logits [rows][world * Vl] (vocab-parallel lm_head)
__global__ void unshard_logits_kernel(const float4* __restrict__ g, float4* __restrict__ out, int world, int rows,
                                      int vl4) {
  griddep_wait();
  griddep_launch();
  const long n = (long)world * rows * vl4;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i % vl4);
    const long rr = i / vl4;
    const int r = (int)(rr % rows), w = (int)(rr / rows);
    out[((long)r * world + w) * vl4 + c] = g[i];
  }
}

int launch_unshard_logits(const float* gathered, float* logits, int world, int rows, int vl, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (vl % 4) return SB_EUNSUPPORTED;
  const long n = (long)world * rows * (vl / 4);
  return launch_k(unshard_logits_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, (const float4*)gathered,
                  (float4*)logits, world, rows, vl / 4);
}

}  // namespace sb
