// Token-level kernels of one speculative iteration:
//   argmax / softmax rows, draft token selection (K1 tail), acceptance (K4),
//   commit + in-place KV rollback (K5), iteration staging + counter RNG.
//
// Semantics follow the reference engine (pkg/src/specbatch/engine.py):
//   verify()        = longest common prefix                     (engine.py:74-86)
//   decode_step()   advanced = min(accepted + 1, remaining)      (engine.py:167)
//                   tokens appended = the verifier's stream      (engine.py:168-171)
//   run_batch()     formed batch held, finished rows masked      (engine.py:186-188)
//   TraceSampler    l = min(trace[I], s), I uniform              (engine.py:109-118)
// The stochastic mode is standard speculative sampling (Leviathan/Chen, cited
// by PAPER.md:43): accept d_j iff u_j * q_j(d_j) < p_j(d_j) (fp32 product),
// else resample from max(0, p_j - q_j); if all k accepted, sample the bonus
// from p_k.  Sampling is a canonical inverse CDF over EXACT fixed-point sums:
// every weight w in [0, 1] becomes the integer W = floor(w * 2^80) (exact from
// the fp32 bits for w >= 2^-57), the pick is the first index v whose inclusive
// prefix P_v satisfies P_v * 2^32 > floor(u * 2^32) * total.  Integer sums are
// associative, so the block computes them in any parallel order and still
// reproduces oracle/spec_ref.py's draw bit for bit.
#include <climits>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace sb {

// -------------------------------------------------------------- row reductions
__device__ ArgMax block_argmax_row(const float* __restrict__ row, int V) {
  ArgMax best{-INFINITY, INT_MAX};
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    float x = row[v];
    if (x > best.v || (x == best.v && v < best.i)) best = ArgMax{x, v};
  }
  best = warp_argmax(best);
  __shared__ float sv[32];
  __shared__ int si[32];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) {
    sv[w] = best.v;
    si[w] = best.i;
  }
  __syncthreads();
  if (w == 0) {
    ArgMax a = lane < nw ? ArgMax{sv[lane], si[lane]} : ArgMax{-INFINITY, INT_MAX};
    a = warp_argmax(a);
    if (lane == 0) {
      sv[0] = a.v;
      si[0] = a.i;
    }
  }
  __syncthreads();
  ArgMax r{sv[0], si[0]};
  __syncthreads();
  return r;
}

__device__ float block_reduce(float v, bool is_max) {
  __shared__ float red[32];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  v = is_max ? warp_max(v) : warp_sum(v);
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    float a = lane < nw ? red[lane] : (is_max ? -INFINITY : 0.f);
    a = is_max ? warp_max(a) : warp_sum(a);
    if (lane == 0) red[0] = a;
  }
  __syncthreads();
  float r = red[0];
  __syncthreads();
  return r;
}

// probs[v] = exp(x[v] - max) / sum  (fp32); in-place allowed
__device__ void block_softmax_row(const float* x, float* p, int V) {
  float m = -INFINITY;
  for (int v = threadIdx.x; v < V; v += blockDim.x) m = fmaxf(m, x[v]);
  m = block_reduce(m, true);
  float s = 0.f;
  for (int v = threadIdx.x; v < V; v += blockDim.x) s += expf(x[v] - m);
  s = block_reduce(s, false);
  float inv = 1.f / s;
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) p[v] = expf(x[v] - m) * inv;
  __syncthreads();
}

// Canonical inverse CDF over weights w[v] = f(v) in [0, 1] (fp32), exact fixed point.
// Mode 0: w = a[v].  Mode 1: w = max(a[v] - b[v], 0).  Returns the index, or -1 if
// every weight is 0.  Thread t owns the contiguous range [t*n, (t+1)*n); range sums
// are exclusive-scanned across the block (128-bit integers: any order is exact); the
// one thread whose range holds the crossing walks it (<= n integer adds).
typedef unsigned __int128 u128;

__device__ __forceinline__ u128 fix80(float w) {
  const uint32_t bits = __float_as_uint(w);
  if ((int32_t)bits <= 0) return 0;        // +0, -0 and negatives
  const uint32_t e = bits >> 23;           // biased exponent (sign bit is 0 here)
  if (e >= 0xFF) return 0;                 // inf / NaN never count
  if (e >= 127) return (u128)1 << 80;      // weights are probabilities: clamp at 1
  if (e == 0) return 0;                    // subnormal (< 2^-126): below the 2^-80 resolution
  const u128 m = (bits & 0x7FFFFF) | 0x800000;
  return e >= 70 ? m << (e - 70) : m >> (70 - e);  // floor(m * 2^(e - 150) * 2^80)
}

__device__ __forceinline__ u128 shfl_up_u128(u128 v, int d) {
  const uint64_t lo = __shfl_up_sync(0xffffffffu, (unsigned long long)(uint64_t)v, d);
  const uint64_t hi = __shfl_up_sync(0xffffffffu, (unsigned long long)(uint64_t)(v >> 64), d);
  return ((u128)hi << 64) | lo;
}

__device__ int block_inverse_cdf(const float* a, const float* b, int mode, int V, float u) {
  __shared__ u128 wsum[32];
  __shared__ u128 total_s;
  __shared__ int pick;
  const int nt = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int n = (V + nt - 1) / nt;
  const int v0 = min(V, t * n), v1 = min(V, v0 + n);
  u128 mine = 0;
  for (int v = v0; v < v1; ++v) mine += fix80(mode ? fmaxf(a[v] - b[v], 0.f) : a[v]);
  // inclusive warp scan, then warp totals
  u128 inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u128 o = shfl_up_u128(inc, d);
    if (lane >= d) inc += o;
  }
  if (t == 0) pick = -1;
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (t == 0) {
    u128 run = 0;
    for (int i = 0; i < (nt >> 5); ++i) {
      const u128 x = wsum[i];
      wsum[i] = run;
      run += x;
    }
    total_s = run;
  }
  __syncthreads();
  const u128 total = total_s;
  if (total != 0) {
    const u128 excl = wsum[w] + inc - mine;
    const u128 target = (u128)(uint64_t)(u * 4294967296.0f) * total;  // floor(u * 2^32) * total < 2^128
    if (mine != 0 && (excl << 32) <= target && ((excl + mine) << 32) > target) {
      u128 run = excl;
      for (int v = v0; v < v1; ++v) {
        run += fix80(mode ? fmaxf(a[v] - b[v], 0.f) : a[v]);
        if ((run << 32) > target) {
          pick = v;
          break;
        }
      }
    }
  }
  __syncthreads();
  const int r = pick;
  __syncthreads();
  return r;
}

// ------------------------------------------------------- cluster-parallel rows
// A vocabulary row (32000-50272 floats) on ONE 256-thread CTA was a serial latency chain: 70-113 us
// per softmax / sample (ncu, stochastic iteration at b=1, k=8: 1.06 ms of 4.15).  Here a cluster of
// RC CTAs owns one row, each CTA a contiguous slice: block reductions, then the RC partials are read
// over DSMEM in rank order (every CTA gets the identical max / sum / total), and the inverse CDF's
// exact fixed-point prefix crosses CTAs through the same exchange.
constexpr int RC = 8;

__device__ __forceinline__ void row_slice(int V, int r, int& lo, int& hi) {
  const int per = ((V + RC - 1) / RC + 3) & ~3;
  lo = min(V, r * per);
  hi = min(V, lo + per);
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ float dsmem_f32(const float* local, int rank) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(dsmem_addr(local, rank)) : "memory");
  return v;
}
__device__ __forceinline__ int dsmem_i32(const int* local, int rank) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(dsmem_addr(local, rank)) : "memory");
  return v;
}
__device__ __forceinline__ u128 dsmem_u128(const u128* local, int rank) {
  unsigned long long lo, hi;
  const uint32_t a = dsmem_addr(local, rank);
  asm volatile("ld.shared::cluster.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(a) : "memory");
  return ((u128)hi << 64) | lo;
}

struct RowSmem {
  float mx, sum;
  float amv;
  int ami;
  u128 tot[2];  // fixed-point slice totals (two inverse-CDF rounds)
  int pick;
};

// Cluster softmax of row x into p (this CTA's slice [lo, hi)): p = expf(x - max) * (1 / sum).
__device__ void cluster_softmax_slice(const float* x, float* p, int lo, int hi, RowSmem& rs) {
  float m = -INFINITY;
  for (int v = lo + threadIdx.x; v < hi; v += blockDim.x) m = fmaxf(m, x[v]);
  m = block_reduce(m, true);
  if (threadIdx.x == 0) rs.mx = m;
  cluster_sync_all();
  m = -INFINITY;
#pragma unroll
  for (int r = 0; r < RC; ++r) m = fmaxf(m, dsmem_f32(&rs.mx, r));
  float sl = 0.f;
  for (int v = lo + threadIdx.x; v < hi; v += blockDim.x) sl += expf(x[v] - m);
  sl = block_reduce(sl, false);
  if (threadIdx.x == 0) rs.sum = sl;
  cluster_sync_all();
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < RC; ++r) s += dsmem_f32(&rs.sum, r);
  const float inv = 1.f / s;
  for (int v = lo + threadIdx.x; v < hi; v += blockDim.x) p[v] = expf(x[v] - m) * inv;
  __syncthreads();
}

// Cluster argmax of row x (ties -> lowest index); every CTA returns the row's winner.
__device__ ArgMax cluster_argmax_row(const float* x, int lo, int hi, RowSmem& rs) {
  ArgMax a = block_argmax_row(x + lo, hi - lo);
  if (threadIdx.x == 0) {
    rs.amv = a.v;
    rs.ami = a.i == INT_MAX ? INT_MAX : a.i + lo;
  }
  cluster_sync_all();
  ArgMax best{-INFINITY, INT_MAX};
#pragma unroll
  for (int r = 0; r < RC; ++r) best = argmax_merge(best, ArgMax{dsmem_f32(&rs.amv, r), dsmem_i32(&rs.ami, r)});
  return best;
}

// Canonical inverse CDF of the row (see block_inverse_cdf) over the cluster: the pick if it lies in
// this CTA's slice, else -1; *total_zero tells every CTA whether all weights were 0.
__device__ int cluster_inverse_cdf(const float* a, const float* b, int mode, int lo, int hi, float u, int round,
                                   RowSmem& rs, bool* total_zero) {
  __shared__ u128 wsum[32];
  const int nt = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int len = hi - lo, n = (len + nt - 1) / nt;
  const int v0 = lo + min(len, t * n), v1 = lo + min(len, t * n + n);
  u128 mine = 0;
  for (int v = v0; v < v1; ++v) mine += fix80(mode ? fmaxf(a[v] - b[v], 0.f) : a[v]);
  u128 inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u128 o = shfl_up_u128(inc, d);
    if (lane >= d) inc += o;
  }
  if (t == 0) rs.pick = -1;
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (t == 0) {
    u128 run = 0;
    for (int i = 0; i < (nt >> 5); ++i) {
      const u128 x = wsum[i];
      wsum[i] = run;
      run += x;
    }
    rs.tot[round] = run;
  }
  cluster_sync_all();
  const int crank = (int)cluster_rank();
  u128 total = 0, off = 0;
#pragma unroll
  for (int r = 0; r < RC; ++r) {
    const u128 x = dsmem_u128(&rs.tot[round], r);
    if (r < crank) off += x;
    total += x;
  }
  *total_zero = total == 0;
  if (total != 0) {
    const u128 excl = off + wsum[w] + inc - mine;
    const u128 target = (u128)(uint64_t)(u * 4294967296.0f) * total;
    if (mine != 0 && (excl << 32) <= target && ((excl + mine) << 32) > target) {
      u128 run = excl;
      for (int v = v0; v < v1; ++v) {
        run += fix80(mode ? fmaxf(a[v] - b[v], 0.f) : a[v]);
        if ((run << 32) > target) {
          rs.pick = v;
          break;
        }
      }
    }
  }
  __syncthreads();
  return rs.pick;
}

// grid (RC, rows), cluster (RC, 1, 1)
__global__ void softmax_rows_cluster_kernel(const float* logits, int V, float* probs) {
  griddep_wait();
  griddep_launch();
  __shared__ RowSmem rs;
  int lo, hi;
  row_slice(V, (int)cluster_rank(), lo, hi);
  cluster_softmax_slice(logits + (size_t)blockIdx.y * V, probs + (size_t)blockIdx.y * V, lo, hi, rs);
  cluster_sync_all();  // peers have read this CTA's partials
}

__global__ void select_cluster_kernel(const float* logits, int V, int mode, const float* __restrict__ u, int u_stride,
                                      float* probs, long long probs_stride, int32_t* out_tok, int out_stride,
                                      int32_t* next_ids, int32_t* next_pos, const int32_t* base_pos, int pos_offset) {
  griddep_wait();
  griddep_launch();
  __shared__ RowSmem rs;
  const int r = blockIdx.y;
  int lo, hi;
  row_slice(V, (int)cluster_rank(), lo, hi);
  const float* row = logits + (size_t)r * V;
  int tok = -1;
  bool mine;
  if (mode == SB_SELECT_ARGMAX) {
    tok = cluster_argmax_row(row, lo, hi, rs).i;
    if (probs) cluster_softmax_slice(row, probs + (size_t)r * probs_stride, lo, hi, rs);
    mine = cluster_rank() == 0;
  } else {
    float* p = probs + (size_t)r * probs_stride;
    cluster_softmax_slice(row, p, lo, hi, rs);
    bool zero;
    tok = cluster_inverse_cdf(p, nullptr, 0, lo, hi, u[(size_t)r * u_stride], 0, rs, &zero);
    mine = tok >= 0;
  }
  if (mine && threadIdx.x == 0) {
    if (out_tok) out_tok[(size_t)r * out_stride] = tok;
    if (next_ids) next_ids[r] = tok;
    if (next_pos) next_pos[r] = base_pos[r] + pos_offset;
  }
  cluster_sync_all();
}

// Stochastic acceptance (mode SB_ACCEPT_STOCHASTIC) with the residual / bonus draw over the cluster.
__global__ void accept_stochastic_cluster_kernel(int k, int V, const float* __restrict__ p_probs,
                                                 const float* __restrict__ q_probs, const int32_t* __restrict__ draft_tok,
                                                 int draft_stride, const float* __restrict__ u_acc,
                                                 const float* __restrict__ u_res, int u_stride,
                                                 const int32_t* __restrict__ produced,
                                                 const int32_t* __restrict__ target_len, int32_t* accepted_len,
                                                 int32_t* advanced, int32_t* out_tok) {
  griddep_wait();
  griddep_launch();
  __shared__ RowSmem rs;
  __shared__ int sh_l;
  const int s = blockIdx.y;
  const int32_t* d = draft_tok + (size_t)s * draft_stride;
  if (threadIdx.x < 32) {  // lane j tests draft j (k <= 32); the first rejection ends the run
    const int j = threadIdx.x;
    bool rej = false;
    if (j < k) {
      const int tok = d[j];
      const float pj = p_probs[((size_t)s * (k + 1) + j) * V + tok];
      const float qj = q_probs[((size_t)s * k + j) * V + tok];
      const float uq = u_acc[(size_t)s * u_stride + j] * qj;
      rej = !(uq < pj);
    }
    const unsigned m = __ballot_sync(0xffffffffu, rej);
    if (j == 0) sh_l = m ? __ffs(m) - 1 : k;
  }
  __syncthreads();
  const int l = sh_l;
  int lo, hi;
  row_slice(V, (int)cluster_rank(), lo, hi);
  const float* p = p_probs + ((size_t)s * (k + 1) + l) * V;
  const float u = u_res[(size_t)s * u_stride];
  bool zero = false;
  int next;
  if (l < k) {
    next = cluster_inverse_cdf(p, q_probs + ((size_t)s * k + l) * V, 1, lo, hi, u, 0, rs, &zero);
    if (zero) next = cluster_inverse_cdf(p, nullptr, 0, lo, hi, u, 1, rs, &zero);
  } else {
    next = cluster_inverse_cdf(p, nullptr, 0, lo, hi, u, 0, rs, &zero);
  }
  int32_t* o = out_tok + (size_t)s * (k + 1);
  if (threadIdx.x == 0 && cluster_rank() == 0) {
    const int rem = target_len[s] - produced[s];
    accepted_len[s] = l;
    advanced[s] = rem <= 0 ? 0 : min(l + 1, rem);
    for (int j = 0; j < l; ++j) o[j] = d[j];
    for (int j = l + 1; j <= k; ++j) o[j] = -1;
  }
  if (threadIdx.x == 0 && next >= 0) o[l] = next;
  cluster_sync_all();
}

template <typename... KArgs, typename... Args>
static int launch_rows_cluster(void (*kern)(KArgs...), int rows, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(RC, rows, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = RC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
  if (e != cudaSuccess) return (int)e;
  ++g_kernel_count;
  return 0;
}

__global__ void argmax_rows_kernel(const float* __restrict__ logits, int V, int32_t* __restrict__ out) {
  griddep_wait();
  griddep_launch();
  ArgMax a = block_argmax_row(logits + (size_t)blockIdx.x * V, V);
  if (threadIdx.x == 0) out[blockIdx.x] = a.i;
}

__global__ void softmax_rows_kernel(const float* logits, int V, float* probs) {
  griddep_wait();
  griddep_launch();
  block_softmax_row(logits + (size_t)blockIdx.x * V, probs + (size_t)blockIdx.x * V, V);
}

__global__ void select_kernel(const float* logits, int V, int mode, const float* __restrict__ u, int u_stride,
                              float* probs, long long probs_stride, int32_t* out_tok, int out_stride,
                              int32_t* next_ids, int32_t* next_pos, const int32_t* base_pos, int pos_offset) {
  griddep_wait();
  griddep_launch();
  int r = blockIdx.x;
  const float* row = logits + (size_t)r * V;
  int tok;
  if (mode == SB_SELECT_ARGMAX) {
    tok = block_argmax_row(row, V).i;
    if (probs) block_softmax_row(row, probs + (size_t)r * probs_stride, V);
  } else {
    float* p = probs + (size_t)r * probs_stride;
    block_softmax_row(row, p, V);
    tok = block_inverse_cdf(p, nullptr, 0, V, u[(size_t)r * u_stride]);
  }
  if (threadIdx.x == 0) {
    if (out_tok) out_tok[(size_t)r * out_stride] = tok;
    if (next_ids) next_ids[r] = tok;
    if (next_pos) next_pos[r] = base_pos[r] + pos_offset;
  }
}

// Finalize of the lm_head-fused argmax: one warp per row merges the per-tile
// (value, index) partials (ties -> lowest index, identical to a full argmax).
// One CTA of 256 threads per row: every tile partial is loaded in one round trip (250 tiles for a
// 32000-entry vocabulary), reduced per warp, then across the 8 warps.  argmax_merge is a total order
// (larger value, then lower index), so the result does not depend on the reduction order.
__global__ void argmax_partials_kernel(const float* __restrict__ val, const int* __restrict__ idx, int n_tiles, int rows,
                                       int32_t* out_tok, int out_stride, int32_t* next_ids, int32_t* next_pos,
                                       const int32_t* base_pos, int pos_offset) {
  __shared__ float wv[8];
  __shared__ int wi[8];
  griddep_wait();
  griddep_launch();
  const int r = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ArgMax a{-INFINITY, INT_MAX};
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
    a = argmax_merge(a, ArgMax{val[(size_t)t * rows + r], idx[(size_t)t * rows + r]});
  a = warp_argmax(a);
  if (lane == 0) {
    wv[warp] = a.v;
    wi[warp] = a.i;
  }
  __syncthreads();
  if (warp == 0) {
    a = lane < (int)(blockDim.x >> 5) ? ArgMax{wv[lane], wi[lane]} : ArgMax{-INFINITY, INT_MAX};
    a = warp_argmax(a);
  }
  if (threadIdx.x == 0) {
    if (out_tok) out_tok[(size_t)r * out_stride] = a.i;
    if (next_ids) next_ids[r] = a.i;
    if (next_pos) next_pos[r] = base_pos[r] + pos_offset;
  }
}

int launch_argmax_partials(const float* val, const int* idx, int n_tiles, int rows, int32_t* out_tok, int out_stride,
                           int32_t* next_ids, int32_t* next_pos, const int32_t* base_pos, int pos_offset,
                           cudaStream_t st) {
  if (rows <= 0) return 0;
  return launch_k(argmax_partials_kernel, dim3(rows), dim3(256), 0, st, val, idx, n_tiles, rows, out_tok, out_stride,
                  next_ids, next_pos, base_pos, pos_offset);
}

int launch_select_argmax(const float* logits, int rows, int vocab, int32_t* out_tok, int out_stride, int32_t* next_ids,
                         int32_t* next_pos, const int32_t* base_pos, int pos_offset, cudaStream_t st) {
  if (rows <= 0) return 0;
  return launch_k(select_kernel, dim3(rows), dim3(256), 0, st, logits, vocab, (int)SB_SELECT_ARGMAX,
                  (const float*)nullptr, 0, (float*)nullptr, 0LL, out_tok, out_stride, next_ids, next_pos, base_pos,
                  pos_offset);
}

// ------------------------------------------------------------------ accept (K4)
__global__ void accept_kernel(int mode, int k, int V, const int32_t* __restrict__ target_tok,
                              const float* __restrict__ p_probs, const float* __restrict__ q_probs,
                              const int32_t* __restrict__ draft_tok, int draft_stride, const float* __restrict__ u_acc,
                              const float* __restrict__ u_res, int u_stride, const int32_t* __restrict__ l_inj,
                              const int32_t* __restrict__ produced, const int32_t* __restrict__ target_len,
                              int32_t* accepted_len, int32_t* advanced, int32_t* out_tok) {
  griddep_wait();
  griddep_launch();
  const int s = blockIdx.x;
  const int32_t* d = draft_tok + (size_t)s * draft_stride;
  __shared__ int sh_l;
  int l = 0, next = 0;
  if (mode == SB_ACCEPT_GREEDY || mode == SB_ACCEPT_INJECTED) {
    const int32_t* t = target_tok + (size_t)s * (k + 1);
    if (mode == SB_ACCEPT_GREEDY) {
      while (l < k && d[l] == t[l]) ++l;
    } else {
      l = min(max(l_inj[s], 0), k);
    }
    next = t[l];
  } else {
    if (threadIdx.x < 32) {  // lane j tests draft j (k <= 32); the first rejection ends the run
      const int j = threadIdx.x;
      bool rej = false;
      if (j < k) {
        const int tok = d[j];
        const float pj = p_probs[((size_t)s * (k + 1) + j) * V + tok];
        const float qj = q_probs[((size_t)s * k + j) * V + tok];
        const float uq = u_acc[(size_t)s * u_stride + j] * qj;
        rej = !(uq < pj);
      }
      const unsigned m = __ballot_sync(0xffffffffu, rej);
      if (j == 0) sh_l = m ? __ffs(m) - 1 : k;
    }
    __syncthreads();
    l = sh_l;
    const float* p = p_probs + ((size_t)s * (k + 1) + l) * V;
    float u = u_res[(size_t)s * u_stride];
    if (l < k) {
      const float* q = q_probs + ((size_t)s * k + l) * V;
      next = block_inverse_cdf(p, q, 1, V, u);
      if (next < 0) next = block_inverse_cdf(p, nullptr, 0, V, u);
    } else {
      next = block_inverse_cdf(p, nullptr, 0, V, u);
    }
  }
  if (threadIdx.x == 0) {
    int rem = target_len[s] - produced[s];
    int adv = rem <= 0 ? 0 : min(l + 1, rem);
    accepted_len[s] = l;
    advanced[s] = adv;
    int32_t* o = out_tok + (size_t)s * (k + 1);
    for (int j = 0; j < l; ++j) o[j] = d[j];
    o[l] = next;
    for (int j = l + 1; j <= k; ++j) o[j] = -1;
  }
}

// ------------------------------------------------------------------ commit (K5)
__global__ void commit_kernel(int b, int k, const int32_t* __restrict__ advanced,
                              const int32_t* __restrict__ accepted_len, const int32_t* __restrict__ out_tok,
                              int32_t* tokens, int cap, int32_t* n_tok, int32_t* produced,
                              const int32_t* __restrict__ target_len, int32_t* finish_iter, int32_t* iter,
                              int32_t* live_count, int32_t* acc_log, int acc_log_cap) {
  griddep_wait();
  griddep_launch();
  __shared__ int live;
  if (threadIdx.x == 0) live = 0;
  __syncthreads();
  const int it = *iter;
  for (int s = threadIdx.x; s < b; s += blockDim.x) {
    int adv = advanced[s];
    bool was_live = produced[s] < target_len[s];
    if (adv > 0) {
      int n = n_tok[s];
      for (int i = 0; i < adv && n + i < cap; ++i) tokens[(size_t)s * cap + n + i] = out_tok[(size_t)s * (k + 1) + i];
      n_tok[s] = n + adv;  // target KV valid length = n_tok - 1: the rejected suffix is rolled back in place
      produced[s] += adv;
    }
    bool live_now = produced[s] < target_len[s];
    if (was_live && !live_now && finish_iter[s] < 0) finish_iter[s] = it + 1;
    if (acc_log && it < acc_log_cap) acc_log[(size_t)it * b + s] = was_live ? accepted_len[s] : -1;
    if (live_now) atomicAdd(&live, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *live_count = live;
    *iter = it + 1;
  }
}

// ------------------------------------------------------------------ staging
__global__ void prepare_kernel(int b, int k, const int32_t* __restrict__ tokens, int cap,
                               const int32_t* __restrict__ n_tok, int32_t* d1_ids, int32_t* d1_pos, int32_t* v_ids,
                               int32_t* v_pos, int32_t* d_last_pos, uint64_t seed, const int32_t* __restrict__ iter,
                               float* uniforms, int n_u, const int32_t* __restrict__ inj, int inj_count,
                               int32_t* l_inj) {
  griddep_wait();
  griddep_launch();
  const uint64_t it = (uint64_t)(*iter);
  for (int s = threadIdx.x; s < b; s += blockDim.x) {
    int n = n_tok[s];
    const int32_t* row = tokens + (size_t)s * cap;
    if (d1_ids) {
      d1_ids[2 * s + 0] = n >= 2 ? row[n - 2] : 0;
      d1_pos[2 * s + 0] = n >= 2 ? n - 2 : -1;
      d1_ids[2 * s + 1] = row[n - 1];
      d1_pos[2 * s + 1] = n - 1;
    }
    v_ids[(size_t)s * (k + 1)] = row[n - 1];
    for (int j = 0; j <= k; ++j) v_pos[(size_t)s * (k + 1) + j] = n - 1 + j;
    if (d_last_pos) d_last_pos[s] = n - 1;
    if (l_inj && inj_count > 0) l_inj[s] = inj[mix3(seed ^ 0x5DEECE66Dull, it, (uint64_t)s) % (uint64_t)inj_count];
  }
  if (uniforms) {
    for (int e = threadIdx.x; e < b * n_u; e += blockDim.x) {
      int s = e / n_u, i = e % n_u;
      uniforms[e] = u01(seed, it, (uint64_t)s * 64 + i);
    }
  }
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_argmax_rows(const float* logits, int32_t rows, int32_t vocab, int32_t* out, void* stream) {
  if (rows <= 0) return 0;
  return launch_k(argmax_rows_kernel, dim3(rows), dim3(256), 0, (cudaStream_t)stream, logits, vocab, out);
}

int sb_softmax_rows(const float* logits, int32_t rows, int32_t vocab, float* probs, void* stream) {
  if (rows <= 0) return 0;
  return launch_rows_cluster(softmax_rows_cluster_kernel, rows, (cudaStream_t)stream, logits, vocab, probs);
}

int sb_select_tokens(const float* logits, int32_t rows, int32_t vocab, int32_t mode, const float* u, int32_t u_stride,
                     float* probs_out, int64_t probs_stride, int32_t* out_tok, int32_t out_stride, int32_t* next_ids,
                     int32_t* next_pos, const int32_t* base_pos, int32_t pos_offset, void* stream) {
  if (rows <= 0) return 0;
  if (mode == SB_SELECT_SAMPLE && (probs_out == nullptr || u == nullptr)) return SB_EINVAL;
  if (next_pos && !base_pos) return SB_EINVAL;
  if (vocab >= 65536) return SB_EUNSUPPORTED;  // fixed-point totals stay below 2^96
  return launch_rows_cluster(select_cluster_kernel, rows, (cudaStream_t)stream, logits, vocab, mode, u, u_stride,
                             probs_out, (long long)probs_stride, out_tok, out_stride, next_ids, next_pos, base_pos,
                             pos_offset);
}

int sb_accept(int32_t mode, int32_t b, int32_t k, int32_t vocab, const int32_t* target_tok, const float* p_probs,
              const float* q_probs, const int32_t* draft_tok, int32_t draft_stride, const float* u_acc,
              const float* u_res, int32_t u_stride, const int32_t* l_inj, const int32_t* produced,
              const int32_t* target_len, int32_t* accepted_len, int32_t* advanced, int32_t* out_tok, void* stream) {
  if (b <= 0 || k < 0 || k > 32) return SB_EINVAL;  // (one warp lane per draft position)
  if (mode == SB_ACCEPT_STOCHASTIC && (!p_probs || (k > 0 && (!q_probs || !u_acc)) || !u_res)) return SB_EINVAL;
  if ((mode == SB_ACCEPT_GREEDY || mode == SB_ACCEPT_INJECTED) && !target_tok) return SB_EINVAL;
  if (mode == SB_ACCEPT_INJECTED && !l_inj) return SB_EINVAL;
  if (mode < 0 || mode > 2) return SB_EINVAL;
  if (vocab >= 65536) return SB_EUNSUPPORTED;  // fixed-point totals stay below 2^96
  if (mode == SB_ACCEPT_STOCHASTIC)
    return launch_rows_cluster(accept_stochastic_cluster_kernel, b, (cudaStream_t)stream, k, vocab, p_probs, q_probs,
                               draft_tok, draft_stride, u_acc, u_res, u_stride, produced, target_len, accepted_len,
                               advanced, out_tok);
  return launch_k(accept_kernel, dim3(b), dim3(256), 0, (cudaStream_t)stream, mode, k, vocab, target_tok, p_probs, q_probs, draft_tok,
                                                     draft_stride, u_acc, u_res, u_stride, l_inj, produced,
                                                     target_len, accepted_len, advanced, out_tok);
}

int sb_kv_commit(int32_t b, int32_t k, const int32_t* advanced, const int32_t* accepted_len, const int32_t* out_tok,
                 int32_t* tokens, int32_t tok_cap, int32_t* n_tok, int32_t* produced, const int32_t* target_len,
                 int32_t* finish_iter, int32_t* iter, int32_t* live_count, int32_t* acc_log, int32_t acc_log_cap,
                 void* stream) {
  if (b <= 0 || k < 0) return SB_EINVAL;
  return launch_k(commit_kernel, dim3(1), dim3(256), 0, (cudaStream_t)stream, b, k, advanced, accepted_len, out_tok, tokens, tok_cap, n_tok,
                                                     produced, target_len, finish_iter, iter, live_count, acc_log,
                                                     acc_log_cap);
}

int sb_prepare_iteration(int32_t b, int32_t k, const int32_t* tokens, int32_t tok_cap, const int32_t* n_tok,
                         int32_t* d1_ids, int32_t* d1_pos, int32_t* v_ids, int32_t* v_pos, int32_t* d_last_pos,
                         uint64_t seed, const int32_t* iter, float* uniforms, int32_t n_u,
                         const int32_t* inj_samples, int32_t inj_count, int32_t* l_inj, void* stream) {
  if (b <= 0 || k < 0 || n_u > 64) return SB_EINVAL;
  if ((d1_ids == nullptr) != (d1_pos == nullptr)) return SB_EINVAL;
  return launch_k(prepare_kernel, dim3(1), dim3(256), 0, (cudaStream_t)stream, b, k, tokens, tok_cap, n_tok, d1_ids, d1_pos, v_ids, v_pos,
                                                      d_last_pos, seed, iter, uniforms, n_u, inj_samples, inj_count,
                                                      l_inj);
}

float sb_uniform_host(uint64_t seed, uint64_t stream_id, uint64_t counter) { return u01(seed, stream_id, counter); }

}  // extern "C"
