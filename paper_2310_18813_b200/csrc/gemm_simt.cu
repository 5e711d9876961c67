// SIMT (FFMA) GEMM: Y[M,N] = X[M,K] . W[N,K]^T with fused epilogues.
//
// This is the fp32 path of the engine ("fp32 greedy output matches the CPU
// reference token for token": tcgen05 has no true-fp32 kind, only tf32) and
// the correctness baseline the tcgen05 kernel is tested against.  Every output
// element is reduced over k in ascending order by one thread, independent of
// M -- the GEMM is batch-invariant, so a position produces bit-identical
// logits whether it is verified in a window of k+1 tokens or decoded alone.
#include "common.cuh"
#include "kernels.cuh"

namespace sb {

constexpr int SBN = 64, SBM = 32, SBK = 32;

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const T* __restrict__ X, const T* __restrict__ W, void* Y,
                                                        int M, int N, int K, int ldx, int epi,
                                                        const T* __restrict__ bias, int relu) {
  __shared__ float Ws[SBK][SBN + 1];
  __shared__ float Xs[SBK][SBM + 1];
  griddep_wait();
  griddep_launch();
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int n_blk = blockIdx.x * SBN, m_blk = blockIdx.y * SBM;
  float acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.f;

  for (int k0 = 0; k0 < K; k0 += SBK) {
    for (int e = tid; e < SBN * SBK; e += 256) {
      int r = e / SBK, kk = e % SBK;
      int n = n_blk + r, k = k0 + kk;
      Ws[kk][r] = (n < N && k < K) ? to_f32(W[(size_t)n * K + k]) : 0.f;
    }
    for (int e = tid; e < SBM * SBK; e += 256) {
      int r = e / SBK, kk = e % SBK;
      int m = m_blk + r, k = k0 + kk;
      Xs[kk][r] = (m < M && k < K) ? to_f32(X[(size_t)m * ldx + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < SBK; ++kk) {
      float w0 = Ws[kk][tx * 4 + 0], w1 = Ws[kk][tx * 4 + 1], w2 = Ws[kk][tx * 4 + 2], w3 = Ws[kk][tx * 4 + 3];
      float x0 = Xs[kk][ty * 2 + 0], x1 = Xs[kk][ty * 2 + 1];
      acc[0][0] = fmaf(w0, x0, acc[0][0]);
      acc[1][0] = fmaf(w1, x0, acc[1][0]);
      acc[2][0] = fmaf(w2, x0, acc[2][0]);
      acc[3][0] = fmaf(w3, x0, acc[3][0]);
      acc[0][1] = fmaf(w0, x1, acc[0][1]);
      acc[1][1] = fmaf(w1, x1, acc[1][1]);
      acc[2][1] = fmaf(w2, x1, acc[2][1]);
      acc[3][1] = fmaf(w3, x1, acc[3][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    int m = m_blk + ty * 2 + j;
    if (m >= M) continue;
    int n0 = n_blk + tx * 4;
    if (epi == EPI_SILU_MUL) {
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        int n = n0 + i;
        if (n + 1 < N) {
          float g = acc[i][j], u = acc[i + 1][j];
          float s = g / (1.f + __expf(-g));
          ((T*)Y)[(size_t)m * (N / 2) + n / 2] = from_f32<T>(s * u);
        }
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int n = n0 + i;
      if (n >= N) continue;
      size_t o = (size_t)m * N + n;
      float v = acc[i][j];
      if (bias) v += to_f32(bias[n]);
      if (relu && epi != EPI_RESID_ADD) v = fmaxf(v, 0.f);
      if (epi == EPI_STORE)
        ((T*)Y)[o] = from_f32<T>(v);
      else if (epi == EPI_STORE_F32)
        ((float*)Y)[o] = v;
      else
        ((float*)Y)[o] += v;
    }
  }
}

int gemm_simt(const GemmArgs& a, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return SB_EINVAL;
  if (a.epi == EPI_ARGMAX || a.ns_part || a.out_part) return SB_EUNSUPPORTED;
  if (a.epi == EPI_SILU_MUL && (a.N & 1)) return SB_EINVAL;
  if (a.epi == EPI_SILU_MUL && (a.bias || a.relu)) return SB_EINVAL;
  dim3 grid((a.N + SBN - 1) / SBN, (a.M + SBM - 1) / SBM);
  if (a.dtype == SB_BF16)
    return launch_k(gemm_simt_kernel<__nv_bfloat16>, grid, dim3(256), 0, st, (const __nv_bfloat16*)a.x,
                    (const __nv_bfloat16*)a.w, a.y, a.M, a.N, a.K, a.ldx, a.epi, (const __nv_bfloat16*)a.bias,
                    a.relu);
  return launch_k(gemm_simt_kernel<float>, grid, dim3(256), 0, st, (const float*)a.x, (const float*)a.w, a.y, a.M, a.N,
                  a.K, a.ldx, a.epi, (const float*)a.bias, a.relu);
}

int g_backend_override = GEMM_AUTO;

int gemm(const GemmArgs& a, int backend, cudaStream_t st) {
  if (backend == GEMM_AUTO) backend = g_backend_override;
  if (backend == GEMM_SIMT) return gemm_simt(a, st);
  if (backend == GEMM_TC) return gemm_tc(a, st);
  if (backend == GEMM_SMALL) return gemm_small(a, st);  // (tests: the draft-step kernel on its own)
  if (a.dtype == SB_BF16 && gemm_tc_supported(a)) return gemm_tc(a, st);
  return gemm_simt(a, st);
}

}  // namespace sb
