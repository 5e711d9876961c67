// Internal launcher declarations (host side).  Each returns 0 or an error code.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "specbatch_b200.h"

namespace sb {

// GEMM epilogues: Y[M,N] = X[M,K] . W[N,K]^T  (fp32 accumulate)
enum GemmEpi : int {
  EPI_STORE = 0,      // y (dtype) [M, N]
  EPI_STORE_F32 = 1,  // y fp32 [M, N]
  EPI_RESID_ADD = 2,  // resid fp32 [M, N] += acc
  EPI_SILU_MUL = 3,   // rows interleaved (gate, up): y (dtype) [M, N/2] = silu(g) * u
  EPI_ARGMAX = 4,     // optional fp32 y [M, N] + per-128-row-tile argmax partials (aux_val/aux_idx [N/128][M])
};

enum GemmBackend : int { GEMM_AUTO = 0, GEMM_SIMT = 1, GEMM_TC = 2, GEMM_SMALL = 3 };

struct GemmArgs {
  int dtype;
  const void* x;  // [M, K] dtype, row stride ldx (elements)
  const void* w;  // [N, K] dtype
  void* y;
  int M, N, K, ldx;
  int epi;
  void* workspace;  // split-K partials / tile counters
  size_t ws_bytes;
  float* aux_val = nullptr;  // EPI_ARGMAX partials
  int* aux_idx = nullptr;
  // fused RMSNorm consumer (tcgen05 only): scale token m by rsqrt(sum_p ns_part[p*ns_stride +
  // m*ns_row_step + ns_row_off] * ns_inv_h + ns_eps); X = bf16(residual * gain), written by the producer
  const float* ns_part = nullptr;
  int ns_P = 0, ns_stride = 0, ns_row_step = 1, ns_row_off = 0;
  float ns_eps = 0.f, ns_inv_h = 0.f;
  // fused RMSNorm producer (EPI_RESID_ADD): bf16 copy of the new residual + sum-of-squares partials
  float* out_part = nullptr;
  void* out_xb = nullptr;
  // RMSNorm gain [N] (bf16) of the consumer of out_xb: out_xb = bf16(new residual * gain); the partials stay
  // sums of new^2, so consumer(xb) * 1/rms == W . (RMSNorm(x) * gain) exactly in real arithmetic
  const void* out_gain = nullptr;
  // OPT: per-output-row bias (model dtype, [N]) added to the fp32 accumulator, then ReLU (store epilogues)
  const void* bias = nullptr;
  int relu = 0;
  // fused LayerNorm (OPT): consumer -- ln_s1 = sums of x partials (layout of ns_part), output row n gets
  // rstd * acc - mean * rstd * ln_c1[n] + ln_c2[n]; producer (EPI_RESID_ADD) -- out_part1 = sums of x
  const float* ln_s1 = nullptr;
  const float* ln_c1 = nullptr;
  const float* ln_c2 = nullptr;
  float* out_part1 = nullptr;
};

extern int g_backend_override;  // sb_set_gemm_backend (ablation / tests)
int gemm(const GemmArgs& a, int backend, cudaStream_t st);
size_t gemm_workspace_bytes(int M, int N, int K);
int gemm_simt(const GemmArgs& a, cudaStream_t st);
int gemm_tc(const GemmArgs& a, cudaStream_t st);  // tcgen05 (bf16 only); SB_EUNSUPPORTED otherwise
bool gemm_tc_supported(const GemmArgs& a);
int gemm_tc_init();
int gemm_tc_norm_partials(const GemmArgs& a);  // rows of out_part this GEMM writes
// small-token GEMM (gemm_small.cu: T <= 16, mma.sync, 16-32 weight rows per CTA); SB_EUNSUPPORTED outside its envelope
extern int g_small_gemm;  // sb_set_small_gemm
bool gemm_small_ok(const GemmArgs& a);
int gemm_small(const GemmArgs& a, cudaStream_t st);
int gemm_small_norm_partials(const GemmArgs& a);  // rows of out_part it writes (one per 16 weight rows)
int gemm_tc_tune(int cps, int stages, int splits);
int gemm_tc_autotune(const void* x, const void* w, float* y, int M, int N, int K, cudaStream_t st, int* cps_out,
                     int* splits_out, float* us_out);
int gemm_tc_autotune_clear();
int gemm_tc_tune_get(int M, int N, int K, int* cps, int* splits, int* wt, int* tn);
int gemm_tc_tune_set(int M, int N, int K, int cps, int splits, int wt, int tn);
int num_sms();
extern int g_w_l2_hint;  // weight-stream L2 policy for the GEMMs of the running forward
// 2-D bf16 tensor map [rows, cols] (row stride ld elements), box TC_BK x box_rows, 128B swizzle.
int make_map(CUtensorMap* map, const void* base, int rows, int cols, int ld, int box_rows);

int launch_embed(int dtype, const void* table, const int32_t* ids, const int32_t* pos, float* h, int n_tok,
                 int hidden, int vocab, cudaStream_t st, const void* pos_table = nullptr, int pos_offset = 0);
int launch_layernorm(int dtype, const float* x, const void* g, const void* b, void* y, int rows, int hidden, float eps,
                     int row_step, int row_off, cudaStream_t st);
int launch_embed_norm(const void* table, const int32_t* ids, const int32_t* pos, float* h, void* xb, float* part,
                      int n_tok, int hidden, int vocab, cudaStream_t st, const void* gain, const void* pos_table = nullptr,
                      int pos_offset = 0, float* part1 = nullptr);
int launch_rmsnorm(int dtype, const float* x, const void* g, void* y, int rows, int hidden, float eps, int row_step,
                   int row_off, cudaStream_t st);
int launch_rope_append(int dtype, const void* qkv, void* q_out, void* kc, void* vc, const int32_t* tok_slot,
                       const int32_t* tok_pos, const float* cosT, const float* sinT, int n_tok, int q_len, int nq,
                       int nkv, int hd, int ctx_max, int max_pos, cudaStream_t st);
int launch_attention(int dtype, const void* q, const void* kc, const void* vc, void* out, const int32_t* tok_slot,
                     const int32_t* tok_pos, int n_seq, int q_len, int nq, int nkv, int hd, int ctx_max,
                     cudaStream_t st);
struct AttnScratch {  // flash-decoding key-split partials (forward workspace)
  float* part;
  float* ml;
  int* counter;  // fixed workspace address, zero between launches
  int max_entries;  // (item, split) partial slots
  int max_items;    // counters
};
extern int g_attn_splits;
int launch_attention_tc(const void* qkv, void* kc, void* vc, void* out, const int32_t* tok_slot, const int32_t* tok_pos,
                        const float* cosT, const float* sinT, int n_seq, int q_len, int nq, int nkv, int hd,
                        int ctx_max, int max_pos, cudaStream_t st, const AttnScratch* scratch = nullptr,
                        const void* l2_next = nullptr, size_t l2_next_bytes = 0);
extern int g_attn_l2pf;
int launch_attention_tc_prefill(const void* qr, void* kc, void* vc, void* out, const int32_t* tok_slot,
                                const int32_t* tok_pos, int n_seq, int q_len, int nq, int nkv, int hd, int ctx_max,
                                cudaStream_t st);
int attention_tc_init();
int launch_argmax_partials(const float* val, const int* idx, int n_tiles, int rows, int32_t* out_tok, int out_stride,
                           int32_t* next_ids, int32_t* next_pos, const int32_t* base_pos, int pos_offset,
                           cudaStream_t st);
int launch_select_argmax(const float* logits, int rows, int vocab, int32_t* out_tok, int out_stride, int32_t* next_ids,
                         int32_t* next_pos, const int32_t* base_pos, int pos_offset, cudaStream_t st);
extern int g_last_count;  // forward.cu: kernels of the last forward / draft loop
int draft_loop_init();     // draft_loop.cu: kernel attributes + co-resident cluster counts (sb_init)
int launch_kv_compact(int dtype, void* k, void* v, const int32_t* src, const int32_t* dst, const int32_t* len, int n,
                      int layers, int slots, int nkv, int ctx_max, int hd, cudaStream_t st);

// ---- tensor-parallel glue (layer_kernels.cu)
int launch_tp_resid_add(float* resid, const void* part, int part_bf16, void* xb, float* npart, int T, int H,
                        cudaStream_t st, const void* gain);
int launch_tp_argmax_pack(const float* val, const int* idx, int n_tiles, int rows, int vocab_off, float* pair,
                          cudaStream_t st);
int launch_tp_argmax_final(const float* pairs, int world, int rows, int32_t* out_tok, int out_stride,
                           int32_t* next_ids, int32_t* next_pos, const int32_t* base_pos, int pos_offset,
                           cudaStream_t st);
int launch_unshard_logits(const float* gathered, float* logits, int world, int rows, int vl, cudaStream_t st);

}  // namespace sb
