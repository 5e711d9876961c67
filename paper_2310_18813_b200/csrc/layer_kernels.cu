// Decoder-layer kernels other than the GEMMs: embedding gather, RMSNorm,
// RoPE + KV append, and KV-cache attention with the causal mask inside the
// speculative window (K3).  All are HBM/latency-bound.
//
// Numerics contract (mirrored by oracle/model_ref.py):
//   residual stream fp32; GEMM inputs rounded to the model dtype after each
//   norm / activation; RoPE applied in fp32 from a host-built fp32 cos/sin
//   table then rounded; attention scores/softmax/accumulation in fp32 with a
//   fixed key order (32-key tiles, ascending) so a query's output does not
//   depend on how many other queries share the launch (batch invariance:
//   spec == greedy exactly in fp32 mode).
#include "common.cuh"
#include "kernels.cuh"

namespace sb {

thread_local int g_kernel_count = 0;

// ---------------------------------------------------------------- embedding
template <typename T>
__global__ void embed_kernel(const T* __restrict__ table, const int32_t* __restrict__ ids,
                             const int32_t* __restrict__ pos, float* __restrict__ h, int hidden, int vocab) {
  int t = blockIdx.x;
  int id = ids[t];
  bool pad = pos != nullptr && pos[t] < 0;
  if (id < 0 || id >= vocab) pad = true;
  const T* row = table + (size_t)(pad ? 0 : id) * hidden;
  float* out = h + (size_t)t * hidden;
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) out[i] = pad ? 0.f : to_f32(row[i]);
}

int launch_embed(int dtype, const void* table, const int32_t* ids, const int32_t* pos, float* h, int n_tok,
                 int hidden, int vocab, cudaStream_t st) {
  if (n_tok <= 0) return 0;
  if (dtype == SB_BF16)
    embed_kernel<__nv_bfloat16><<<n_tok, 256, 0, st>>>((const __nv_bfloat16*)table, ids, pos, h, hidden, vocab);
  else
    embed_kernel<float><<<n_tok, 256, 0, st>>>((const float*)table, ids, pos, h, hidden, vocab);
  g_kernel_count++;
  SB_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------- RMSNorm
// y[r] = dtype(x[src_row(r)] * rsqrt(mean(x^2) + eps) * g); src_row(r) = r*row_step + row_off
template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x, const T* __restrict__ g,
                                                      T* __restrict__ y, int hidden, float eps, int row_step,
                                                      int row_off) {
  int r = blockIdx.x;
  const float* xr = x + (size_t)(r * row_step + row_off) * hidden;
  float ss = 0.f;
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) {
    float v = xr[i];
    ss += v * v;
  }
  __shared__ float red[8];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  float inv = rsqrtf(red[0] / (float)hidden + eps);
  T* yr = y + (size_t)r * hidden;
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) yr[i] = from_f32<T>(xr[i] * inv * to_f32(g[i]));
}

int launch_rmsnorm(int dtype, const float* x, const void* g, void* y, int rows, int hidden, float eps, int row_step,
                   int row_off, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (dtype == SB_BF16)
    rmsnorm_kernel<__nv_bfloat16><<<rows, 256, 0, st>>>(x, (const __nv_bfloat16*)g, (__nv_bfloat16*)y, hidden, eps,
                                                        row_step, row_off);
  else
    rmsnorm_kernel<float><<<rows, 256, 0, st>>>(x, (const float*)g, (float*)y, hidden, eps, row_step, row_off);
  g_kernel_count++;
  SB_CHECK_LAUNCH();
  return 0;
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
  int t = blockIdx.x;
  int slot = tok_slot[t / q_len];
  int p = tok_pos[t];
  int half = hd / 2;
  const T* row = qkv + (size_t)t * (nq + 2 * nkv) * hd;
  int pc = p < 0 ? 0 : (p >= max_pos ? max_pos - 1 : p);
  const float* cr = cosT + (size_t)pc * half;
  const float* sr = sinT + (size_t)pc * half;
  // q heads
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

int launch_rope_append(int dtype, const void* qkv, void* q_out, void* kc, void* vc, const int32_t* tok_slot,
                       const int32_t* tok_pos, const float* cosT, const float* sinT, int n_tok, int q_len, int nq,
                       int nkv, int hd, int ctx_max, int max_pos, cudaStream_t st) {
  if (n_tok <= 0) return 0;
  if (dtype == SB_BF16)
    rope_append_kernel<__nv_bfloat16><<<n_tok, 256, 0, st>>>(
        (const __nv_bfloat16*)qkv, (__nv_bfloat16*)q_out, (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, tok_slot, tok_pos,
        cosT, sinT, q_len, nq, nkv, hd, ctx_max, max_pos);
  else
    rope_append_kernel<float><<<n_tok, 256, 0, st>>>((const float*)qkv, (float*)q_out, (float*)kc, (float*)vc,
                                                     tok_slot, tok_pos, cosT, sinT, q_len, nq, nkv, hd, ctx_max,
                                                     max_pos);
  g_kernel_count++;
  SB_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------- attention (K3)
// One CTA per (q head, sequence, query group of kQG).  Keys of the slot are
// streamed in 32-key tiles (coalesced loads into padded smem); each
// query j at absolute position p_j sees keys [0, p_j] (causal inside the
// speculative window).  Online softmax in fp32 with a fixed key order
// (32-key tiles, ascending).
constexpr int kAttnKT = 32;   // keys per tile (one per lane)
constexpr int kAttnQG = 16;   // queries per CTA

// HD threads per CTA (thread d owns output dim d); HD/32 warps share the
// score / softmax work.  Supported head dims: 64, 128.
template <typename T, int HD>
__global__ void __launch_bounds__(HD) attention_kernel(const T* __restrict__ q, const T* __restrict__ kc,
                                                        const T* __restrict__ vc, T* __restrict__ out,
                                                        const int32_t* __restrict__ tok_slot,
                                                        const int32_t* __restrict__ tok_pos, int q_len, int nq,
                                                        int nkv, int ctx_max, float scale) {
  constexpr int NW = HD / 32;
  constexpr int KP = HD + 1;  // padded row (floats) -> conflict-free column reads
  __shared__ float Ks[kAttnKT][KP];
  __shared__ float Vs[kAttnKT][HD];
  __shared__ float Qs[kAttnQG][HD];
  __shared__ float S[kAttnQG][kAttnKT];
  __shared__ float m_run[kAttnQG], l_run[kAttnQG], corr[kAttnQG];

  const int head = blockIdx.x, seq = blockIdx.y, qg = blockIdx.z;
  const int kvh = head / (nq / nkv);
  const int slot = tok_slot[seq];
  const int tid = threadIdx.x;
  const int j0 = qg * kAttnQG;
  const int nqg = min(kAttnQG, q_len - j0);
  if (nqg <= 0) return;

  int maxp = -1;
  for (int j = 0; j < nqg; ++j) maxp = max(maxp, tok_pos[seq * q_len + j0 + j]);

  for (int e = tid; e < kAttnQG * HD; e += HD) {
    int j = e / HD, d = e % HD;
    float v = 0.f;
    if (j < nqg) v = to_f32(q[((size_t)(seq * q_len + j0 + j) * nq + head) * HD + d]) * scale;
    Qs[j][d] = v;
  }
  if (tid < kAttnQG) {
    m_run[tid] = -INFINITY;
    l_run[tid] = 0.f;
  }
  float acc[kAttnQG];
#pragma unroll
  for (int j = 0; j < kAttnQG; ++j) acc[j] = 0.f;

  const T* kbase = kc + ((size_t)slot * nkv + kvh) * ctx_max * HD;
  const T* vbase = vc + ((size_t)slot * nkv + kvh) * ctx_max * HD;
  const int n_keys = maxp + 1;
  __syncthreads();

  for (int k0 = 0; k0 < n_keys; k0 += kAttnKT) {
    const int nk = min(kAttnKT, n_keys - k0);
    for (int e = tid; e < kAttnKT * HD; e += HD) {
      int r = e / HD, d = e % HD;
      float kv = 0.f, vv = 0.f;
      if (r < nk) {
        kv = to_f32(kbase[(size_t)(k0 + r) * HD + d]);
        vv = to_f32(vbase[(size_t)(k0 + r) * HD + d]);
      }
      Ks[r][d] = kv;
      Vs[r][d] = vv;
    }
    __syncthreads();
    // scores: thread handles key r = lane for queries j = warp, warp+4, ...
    {
      int r = tid & (kAttnKT - 1);
      for (int j = tid >> 5; j < kAttnQG; j += NW) {
        float s = -INFINITY;
        if (j < nqg) {
          int pj = tok_pos[seq * q_len + j0 + j];
          if (r < nk && k0 + r <= pj) {
            float a = 0.f;
#pragma unroll 16
            for (int d = 0; d < HD; ++d) a = fmaf(Qs[j][d], Ks[r][d], a);
            s = a;
          }
        }
        S[j][r] = s;
      }
    }
    __syncthreads();
    // online softmax update: warp w handles queries w, w+4, ...
    {
      int w = tid >> 5, lane = tid & 31;
      for (int j = w; j < kAttnQG; j += NW) {
        float a = S[j][lane];
        float mt = warp_max(a);
        float mo = m_run[j];
        float mn = fmaxf(mo, mt);
        float ea = (mn == -INFINITY) ? 0.f : __expf(a - mn);
        S[j][lane] = ea;
        float sum = warp_sum(ea);
        if (lane == 0) {
          float c = (mo == -INFINITY) ? 0.f : __expf(mo - mn);
          corr[j] = c;
          l_run[j] = l_run[j] * c + sum;
          m_run[j] = mn;
        }
      }
    }
    __syncthreads();
    // P.V: thread owns output dim d = tid for all queries
    {
      int d = tid;
#pragma unroll
      for (int j = 0; j < kAttnQG; ++j) acc[j] *= corr[j];
      for (int r = 0; r < nk; ++r) {
        float vv = Vs[r][d];
#pragma unroll
        for (int j = 0; j < kAttnQG; ++j) acc[j] = fmaf(S[j][r], vv, acc[j]);
      }
    }
    __syncthreads();
  }
  for (int j = 0; j < nqg; ++j) {
    float l = l_run[j];
    float o = l > 0.f ? acc[j] / l : 0.f;
    out[((size_t)(seq * q_len + j0 + j) * nq + head) * HD + tid] = from_f32<T>(o);
  }
}

int launch_attention(int dtype, const void* q, const void* kc, const void* vc, void* out, const int32_t* tok_slot,
                     const int32_t* tok_pos, int n_seq, int q_len, int nq, int nkv, int hd, int ctx_max,
                     cudaStream_t st) {
  if ((hd != 64 && hd != 128) || nq % nkv != 0) return SB_EUNSUPPORTED;
  dim3 grid(nq, n_seq, (q_len + kAttnQG - 1) / kAttnQG);
  float scale = 1.0f / sqrtf((float)hd);
#define SB_ATTN(T, HD)                                                                                        \
  attention_kernel<T, HD><<<grid, HD, 0, st>>>((const T*)q, (const T*)kc, (const T*)vc, (T*)out, tok_slot, tok_pos, \
                                               q_len, nq, nkv, ctx_max, scale)
  if (dtype == SB_BF16) {
    if (hd == 128) SB_ATTN(__nv_bfloat16, 128); else SB_ATTN(__nv_bfloat16, 64);
  } else {
    if (hd == 128) SB_ATTN(float, 128); else SB_ATTN(float, 64);
  }
#undef SB_ATTN
  g_kernel_count++;
  SB_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------- KV compaction (K5)
template <typename T>
__global__ void kv_compact_kernel(T* __restrict__ k, T* __restrict__ v, const int32_t* __restrict__ src,
                                  const int32_t* __restrict__ dst, const int32_t* __restrict__ len, int slots,
                                  int nkv, int ctx_max, int hd) {
  int i = blockIdx.y, layer = blockIdx.z;
  int s = src[i], d = dst[i];
  if (s == d) return;
  size_t per = (size_t)len[i] * hd;
  for (int h = 0; h < nkv; ++h) {
    size_t so = (((size_t)layer * slots + s) * nkv + h) * ctx_max * hd;
    size_t doff = (((size_t)layer * slots + d) * nkv + h) * ctx_max * hd;
    for (size_t e = blockIdx.x * blockDim.x + threadIdx.x; e < per; e += (size_t)gridDim.x * blockDim.x) {
      k[doff + e] = k[so + e];
      v[doff + e] = v[so + e];
    }
  }
}

int launch_kv_compact(int dtype, void* k, void* v, const int32_t* src, const int32_t* dst, const int32_t* len, int n,
                      int layers, int slots, int nkv, int ctx_max, int hd, cudaStream_t st) {
  if (n <= 0) return 0;
  dim3 grid(8, n, layers);
  if (dtype == SB_BF16)
    kv_compact_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((__nv_bfloat16*)k, (__nv_bfloat16*)v, src, dst, len, slots,
                                                           nkv, ctx_max, hd);
  else
    kv_compact_kernel<float><<<grid, 256, 0, st>>>((float*)k, (float*)v, src, dst, len, slots, nkv, ctx_max, hd);
  SB_CHECK_LAUNCH();
  return 0;
}

}  // namespace sb
