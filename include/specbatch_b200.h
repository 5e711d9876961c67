/*
 * specbatch_b200.h -- C-ABI of the B200-native batched speculative-decoding engine.
 *
 * The reference (arXiv 2310.18813, package `specbatch`) is pure Python and has
 * no FFI; the drop-in boundary it defines is the per-step oracle/run_batch
 * surface (pkg/src/specbatch/engine.py:100-106, 155-221).  Every entry point
 * below replaces one piece of that step on the GPU and is cited against the
 * reference symbol whose semantics it implements:
 *
 *   sb_decoder_forward   <- the model evaluations hidden behind DraftOracle.step
 *                           (engine.py:100-106; TokenLevel.target_token /
 *                           draft_tokens engine.py:135-145): draft step (K1) and
 *                           target verify forward (K2 GEMMs + K3 attention)
 *   sb_select_tokens     <- greedy argmax / sampling of the next token
 *                           (TokenLevel.draft_tokens engine.py:138-145)
 *   sb_accept            <- verify() LCP (engine.py:74-86) + decode_step's
 *                           advanced = min(accepted+1, remaining) (engine.py:167);
 *                           stochastic min(1,p/q) mode (PAPER.md:43 refs) (K4)
 *   sb_kv_commit         <- state.produced += advanced; tokens.extend
 *                           (engine.py:168-172) + in-place KV rollback (K5)
 *   sb_kv_compact        <- (new) slab compaction when sequences retire (K5)
 *   sb_prepare_*         <- per-iteration input staging (no reference analogue;
 *                           keeps every iteration graph-replayable)
 *
 * Conventions: every call is asynchronous on `stream`, graph-capturable, does
 * not allocate, takes caller-owned device buffers and returns 0 on success or
 * a cudaError_t / SB_E* code.  No torch types cross this boundary.
 */
#ifndef SPECBATCH_B200_H
#define SPECBATCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB_ABI_VERSION 10

/* status codes beyond cudaError_t (which are < 1000) */
#define SB_OK 0
#define SB_EINVAL 1001      /* bad shape / argument (maps to ValueError) */
#define SB_EWORKSPACE 1002  /* workspace too small */
#define SB_EUNSUPPORTED 1003

/* dtypes */
#define SB_BF16 0
#define SB_F32 1

/* decoder architectures (sb_decoder_t.arch) */
#define SB_ARCH_LLAMA 0 /* RMSNorm, RoPE, SwiGLU, GQA, untied lm_head (Llama-2, LLaMA-68M/160M) */
#define SB_ARCH_OPT 1   /* LayerNorm+bias, learned positions (+offset), biased projections, ReLU FFN, tied head */

/* logits selection for sb_decoder_forward */
#define SB_LOGITS_ALL 0   /* one logits row per input token                */
#define SB_LOGITS_LAST 1  /* one row per sequence (its last query token)   */
#define SB_LOGITS_NONE 2  /* prefill: KV only                              */

/* acceptance modes for sb_accept */
#define SB_ACCEPT_GREEDY 0     /* LCP of draft vs target argmax               */
#define SB_ACCEPT_STOCHASTIC 1 /* u*q(d) < p(d); residual resample            */
#define SB_ACCEPT_INJECTED 2   /* l = min(l_inj, k): TraceSampler law on device */

/* token selection modes for sb_select_tokens */
#define SB_SELECT_ARGMAX 0
#define SB_SELECT_SAMPLE 1

/*
 * Tensor-parallel exchange (BASELINE config 4: a target too large for one GPU,
 * sharded over 2/4/8 GPUs of one NVLink box).  The forward calls these at its
 * two exchange points per layer (after the row-parallel o / down projections:
 * all_reduce_sum of the fp32 partial residual update) and once for the
 * vocab-parallel lm_head (all_gather of the local logits slice).  Both are
 * asynchronous on `stream`.  sb_nccl_collectives_init fills one backed by NCCL
 * over NVLink (graph-capturable); a host may supply its own (tests use
 * torch.distributed gloo to run TP=2 on one GPU).  Return 0 or an error code.
 */
typedef struct sb_collectives {
  void* ctx;
  int (*all_reduce_sum)(void* ctx, void* buf, size_t count, int32_t dtype, void* stream);
  int (*all_gather)(void* ctx, const void* send, void* recv, size_t count_per_rank, int32_t dtype, void* stream);
  int32_t world, rank;
} sb_collectives_t;

/* NCCL backend: rank 0 makes the 128-byte id, the host broadcasts it, every rank inits. */
int sb_nccl_unique_id(void* id_out);
int sb_nccl_collectives_init(const void* id, int32_t world, int32_t rank, sb_collectives_t* out);
int sb_nccl_collectives_destroy(sb_collectives_t* c);

/*
 * Llama-style decoder weights.  Arrays of per-layer DEVICE pointers are host
 * arrays (read by the launcher).  Layouts (row-major, K contiguous):
 *   embed      [vocab, hidden]
 *   w_qkv[l]   [(n_heads + 2*n_kv_heads)*head_dim, hidden]  rows: Q | K | V
 *   w_o[l]     [hidden, n_heads*head_dim]
 *   w_gu[l]    [2*ffn, hidden]  rows interleaved g0,u0,g1,u1,...
 *   w_down[l]  [hidden, ffn]
 *   lm_head    [vocab, hidden]
 *   norms      [hidden] in `dtype`: RMSNorm gains attn_norm[l] (before qkv),
 *              mlp_norm[l] (before gate/up), final_norm (before lm_head).
 *              Applied as y = x / rms(x) * g on every path: the fp32 path
 *              materialises the normalised row; the bf16 path fuses the norm
 *              into the GEMMs -- the producer of the residual (embedding,
 *              o_proj, down_proj, TP reduce) writes xb = bf16(x * g_next) and
 *              per-tile sums of x^2, the consumer GEMM scales its output
 *              row by 1/rms.  Gains are NOT folded into the weights.
 *   rope_cos/rope_sin [max_pos, head_dim/2] fp32 (host-computed table)
 */
typedef struct sb_decoder {
  int32_t n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab;
  int32_t dtype;   /* SB_BF16 | SB_F32 */
  int32_t max_pos; /* rows of the rope table */
  float rms_eps;
  const void* embed;
  const void* final_norm;
  const void* lm_head;
  const void* const* attn_norm;
  const void* const* w_qkv;
  const void* const* w_o;
  const void* const* mlp_norm;
  const void* const* w_gu;
  const void* const* w_down;
  const float* rope_cos;
  const float* rope_sin;
  /* tensor parallelism (NULL = unsharded).  A shard holds n_heads/world q heads,
     n_kv_heads/world kv heads, ffn/world ffn rows and vocab/world lm_head rows
     (the fields above are the LOCAL sizes); embedding and norms are replicated.
     Logits come back full-width [rows, vocab * world] on every rank. */
  const sb_collectives_t* tp;
  /* SB_ARCH_OPT (BASELINE config 2: OPT-125M / OPT-6.7B).  For OPT, w_gu holds
     fc1 [ffn, hidden] (no gate) and w_down fc2 [hidden, ffn]; attn_norm /
     mlp_norm / final_norm are LayerNorm gains with the *_b betas; lm_head may
     alias embed (tied); the rope tables are identity (cos 1, sin 0). */
  int32_t arch;
  int32_t pos_offset;             /* learned position p reads pos_embed row p + pos_offset (OPT: 2) */
  const void* pos_embed;          /* [max_pos + pos_offset, hidden] */
  const void* final_norm_b;
  const void* const* attn_norm_b;
  const void* const* mlp_norm_b;
  const void* const* b_qkv;       /* [(n_heads + 2 n_kv_heads) head_dim] */
  const void* const* b_o;         /* [hidden] */
  const void* const* b_fc1;       /* [ffn] */
  const void* const* b_fc2;       /* [hidden] */
  /* OPT, bf16: LayerNorm fused into the consuming GEMMs (all NULL = separate LayerNorm kernels).  For a
     consumer with weight W [N, K] behind LayerNorm (gamma, beta): c1 = W gamma, c2 = W beta (fp32 [N]),
     and W . LN(x) = rstd * W . (x * gamma) - mean * rstd * c1 + c2, with the residual's producer writing
     xb = bf16(x * gamma) and per-tile sums of x and x^2 (mean, rstd in the consumer's epilogue). */
  const float* const* ln_qkv_c1;  /* [n_layers] -> [qkv rows] */
  const float* const* ln_qkv_c2;
  const float* const* ln_fc1_c1;  /* [n_layers] -> [ffn] */
  const float* const* ln_fc1_c2;
  const float* ln_lm_c1;          /* [vocab] */
  const float* ln_lm_c2;
  /* 1 = a draft model: its decode-sized bf16 GEMMs (<= 16 tokens, <= 8M weights) may take the small-token
     kernel (sb_set_small_gemm).  0 (targets) keeps one GEMM kernel family across token counts, so a greedy
     verify of k+1 tokens computes what k+1 single-token decodes would. */
  int32_t role;
} sb_decoder_t;

/* KV cache: k/v base pointers of layout [n_layers][slots][n_kv_heads][ctx_max][head_dim]. */
typedef struct sb_kvcache {
  void* k;
  void* v;
  int32_t slots, ctx_max;
} sb_kvcache_t;

/* Workspace bytes sb_decoder_forward needs for n_tokens query tokens. */
size_t sb_decoder_workspace_bytes(const sb_decoder_t* m, int32_t n_tokens);

/*
 * One forward of a uniform-q_len batch: n_seq sequences x q_len tokens
 * (token t = s*q_len + j).  tok_slot[s] is the KV slot of sequence s;
 * tok_pos[t] the absolute position (-1 = padding: no KV write, masked).
 * Query at position p attends keys [0, p] of its slot (causal inside the
 * speculative window).  logits fp32: [n_tok or n_seq, vocab].
 */
int sb_decoder_forward(const sb_decoder_t* m, const sb_kvcache_t* kv, const int32_t* tok_ids,
                       const int32_t* tok_slot, const int32_t* tok_pos, int32_t n_seq, int32_t q_len,
                       float* logits, int32_t logits_mode, void* workspace, size_t ws_bytes,
                       void* stream);

/*
 * Greedy token sink: when passed to sb_decoder_forward_ex, the argmax of every
 * logits row (ties -> lowest index) is computed inside the lm_head GEMM
 * epilogue (per-128-row partials + one-warp finalize) and written to
 * out_tok[r*out_stride], next_ids[r], next_pos[r] = base_pos[r] + pos_offset
 * (each pointer optional).  logits may then be NULL (not materialised).
 */
typedef struct sb_token_sink {
  int32_t* out_tok;
  int32_t out_stride;
  int32_t* next_ids;
  int32_t* next_pos;
  const int32_t* base_pos;
  int32_t pos_offset;
} sb_token_sink_t;

int sb_decoder_forward_ex(const sb_decoder_t* m, const sb_kvcache_t* kv, const int32_t* tok_ids,
                          const int32_t* tok_slot, const int32_t* tok_pos, int32_t n_seq, int32_t q_len,
                          float* logits, int32_t logits_mode, const sb_token_sink_t* sink, void* workspace,
                          size_t ws_bytes, void* stream);

/*
 * Verify windows plus riding prompts in ONE forward (continuous batching:
 * prompts admitted into freed slots are prefilled inside the next verify
 * instead of by a separate weight stream).  tok_ids / tok_pos hold the
 * n_seq x q_len window tokens (KV slots tok_slot[n_seq]) followed by pf_n
 * prompts of pf_len tokens (KV slots pf_slot[pf_n]); every token shares the
 * GEMMs, the prompts get their own attention launch and no logits: logits /
 * sink cover the window rows exactly as sb_decoder_forward_ex.  Workspace:
 * sb_decoder_workspace_bytes(n_seq*q_len + pf_n*pf_len).  Llama bf16
 * (unsharded) only, else SB_EUNSUPPORTED.  Reference: the reference has no
 * prefill; SURVEY 8(f)2 / 8(f)4.
 */
int sb_decoder_forward_mixed(const sb_decoder_t* m, const sb_kvcache_t* kv, const int32_t* tok_ids,
                             const int32_t* tok_slot, const int32_t* tok_pos, int32_t n_seq, int32_t q_len,
                             int32_t pf_n, int32_t pf_len, const int32_t* pf_slot, float* logits,
                             int32_t logits_mode, const sb_token_sink_t* sink, void* workspace, size_t ws_bytes,
                             void* stream);

/*
 * Next-token selection over logits rows [rows, vocab] (fp32).
 *   ARGMAX: ties -> lowest index (np.argmax); probs_out optional.
 *   SAMPLE: probs_out[r*probs_stride + v] = softmax(logits[r]) (fp32), token =
 *           canonical exact inverse CDF at u[r*u_stride] (see sb_accept).
 * Token r is written to out_tok[r*out_stride] (if non-NULL), next_ids[r], and
 * next_pos[r] = base_pos[r] + pos_offset (staging the next draft step).
 * Reference: TokenLevel.draft_tokens (engine.py:138-145) -- here the draft is
 * a real model and the token is its argmax / sample.
 */
int sb_select_tokens(const float* logits, int32_t rows, int32_t vocab, int32_t mode, const float* u,
                     int32_t u_stride, float* probs_out, int64_t probs_stride, int32_t* out_tok,
                     int32_t out_stride, int32_t* next_ids, int32_t* next_pos, const int32_t* base_pos,
                     int32_t pos_offset, void* stream);

/* Row softmax: probs[r] = softmax(logits[r]) (fp32, max-subtracted); in place allowed. */
int sb_softmax_rows(const float* logits, int32_t rows, int32_t vocab, float* probs, void* stream);

/* Row argmax (ties -> lowest index). */
int sb_argmax_rows(const float* logits, int32_t rows, int32_t vocab, int32_t* out, void* stream);

/*
 * Acceptance (K4) for b sequences at speculation length k (>= 0).
 *   target_tok [b, k+1]      target argmax per verify position (GREEDY / INJECTED)
 *   p_probs    [b, k+1, V]   target probabilities (STOCHASTIC)
 *   q_probs    [b, k, V]     draft probabilities (STOCHASTIC)
 *   draft_tok  row s at draft_tok + s*draft_stride, k entries
 *   u_acc[s*u_stride + j], u_res[s*u_stride]  uniforms in [0,1) (STOCHASTIC)
 *   l_inj [b]                injected accepted lengths (INJECTED)
 *   produced/target_len [b]  remaining = target_len - produced (<= 0: finished, masked)
 * GREEDY:     l = LCP(draft, target_tok[:k])          (verify, engine.py:74-86)
 * INJECTED:   l = min(l_inj, k)                        (TraceSampler, engine.py:109-118)
 * STOCHASTIC: accept d_j iff fp32(u_acc_j * q_j(d_j)) < p_j(d_j); on the first
 *             rejection resample from max(0, p_l - q_l), else the bonus from p_k.
 *             One warp lane per draft position (ballot: the first rejection).
 *             Inverse CDF over exact fixed point: W_v = floor(w_v * 2^80) (w in
 *             [0,1] fp32), pick = first v with P_v * 2^32 > floor(u * 2^32) * total
 *             (P_v inclusive prefix; integer sums, so any parallel order is exact
 *             and the oracle reproduces every draw bit for bit).  vocab < 65536.
 * Outputs: accepted_len[b]; advanced[b] = min(l+1, remaining) or 0 if finished
 *          (engine.py:167); out_tok[b, k+1] = d_1..d_l, next, then -1 padding.
 */
int sb_accept(int32_t mode, int32_t b, int32_t k, int32_t vocab, const int32_t* target_tok,
              const float* p_probs, const float* q_probs, const int32_t* draft_tok, int32_t draft_stride,
              const float* u_acc, const float* u_res, int32_t u_stride, const int32_t* l_inj,
              const int32_t* produced, const int32_t* target_len, int32_t* accepted_len, int32_t* advanced,
              int32_t* out_tok, void* stream);

/*
 * Commit (K5): append out_tok[s, :advanced] to tokens[s, tok_cap] at n_tok[s];
 * n_tok += advanced; produced += advanced (engine.py:168-172).  The target
 * KV valid length is n_tok - 1 and the draft re-feeds the last two committed
 * tokens each iteration, so the rejected suffix is rolled back in place: its
 * KV rows are simply overwritten by the next iteration (no copy).
 * finish_iter[s] (init -1) <- 1-based iteration at which s finished;
 * acc_log[iter*b + s] <- accepted_len (-1 once finished) while iter < acc_log_cap;
 * live_count <- #unfinished; iter += 1.
 */
int sb_kv_commit(int32_t b, int32_t k, const int32_t* advanced, const int32_t* accepted_len,
                 const int32_t* out_tok, int32_t* tokens, int32_t tok_cap, int32_t* n_tok, int32_t* produced,
                 const int32_t* target_len, int32_t* finish_iter, int32_t* iter, int32_t* live_count,
                 int32_t* acc_log, int32_t acc_log_cap, void* stream);

/*
 * Stage one iteration from committed state (n = n_tok[s]):
 *   d1_ids/d1_pos [b, 2] = (tokens[n-2], n-2), (tokens[n-1], n-1); pos -1 if n < 2
 *   v_ids[s*(k+1)] = tokens[n-1]; v_pos[s, j] = n-1+j (j = 0..k)
 *   d_last_pos[s] = n-1 (base for sb_select_tokens' next_pos)
 *   uniforms[s*n_u + i] = sb_uniform_host(seed, iter, s*64 + i)   (n_u <= 64)
 *   l_inj[s] = inj_samples[mix(seed ^ 0x5DEECE66D, iter, s) % inj_count]
 * Any output pointer may be NULL (skipped).
 */
int sb_prepare_iteration(int32_t b, int32_t k, const int32_t* tokens, int32_t tok_cap, const int32_t* n_tok,
                         int32_t* d1_ids, int32_t* d1_pos, int32_t* v_ids, int32_t* v_pos,
                         int32_t* d_last_pos, uint64_t seed, const int32_t* iter, float* uniforms,
                         int32_t n_u, const int32_t* inj_samples, int32_t inj_count, int32_t* l_inj,
                         void* stream);

/*
 * The whole greedy draft loop of one iteration in ONE persistent launch (K1),
 * replacing k x (draft forward + token sink) -- the draft proposals of
 * DraftOracle.step / TokenLevel.draft_tokens (engine.py:100-106, 138-145).
 * Steps j = 1..k of the draft decoder for b sequences, staged exactly like k
 * calls of sb_decoder_forward_ex with a token sink: step 1 feeds d1_ids /
 * d1_pos (the last two committed tokens per sequence, [b, 2]), step j >= 2
 * feeds d_{j-1} at position d_base[s] + j - 1; writes v_ids[s*(k+1) + j] = d_j,
 * ds_ids[s] = d_j, ds_pos[s] = d_base[s] + j.  One CTA per SM (thread-block
 * clusters of ffn/hidden CTAs), grid barriers between phases, a producer warp
 * streaming weight tiles ahead of the barriers.  workspace: at least
 * sb_draft_loop_workspace_bytes(m) bytes (contents scratch); sync_words: 64
 * zero-initialised bytes owned by this call site (self-resetting barrier words,
 * never shared with a concurrently running launch).  SB_EUNSUPPORTED outside
 * its envelope (bf16 Llama-arch, unsharded, head_dim 64, 2b <= 16, ffn/hidden
 * in {2,4,8}, hidden <= 1024) or when disabled: the caller then issues the
 * per-step forwards.
 */
int sb_draft_loop(const sb_decoder_t* m, const sb_kvcache_t* kv, const void* packed, int32_t b, int32_t k,
                  const int32_t* d1_ids, const int32_t* d1_pos, const int32_t* slots, const int32_t* d_base,
                  int32_t* v_ids, int32_t* ds_ids, int32_t* ds_pos, void* workspace, size_t ws_bytes,
                  void* sync_words, void* stream);
/* The draft's weights re-laid for sb_draft_loop ("packed"): every 16-row x hidden tile contiguous and
   128B-swizzled so one bulk copy feeds a conflict-free ldmatrix; written by sb_draft_loop_pack (once,
   and again whenever the weights change) into a caller buffer of sb_draft_loop_packed_bytes(m)
   bytes (0 = outside the envelope). */
size_t sb_draft_loop_packed_bytes(const sb_decoder_t* m);
int sb_draft_loop_pack(const sb_decoder_t* m, void* dst, size_t bytes, void* stream);
size_t sb_draft_loop_workspace_bytes(const sb_decoder_t* m);
/* Diagnostics: device buffer (>= 4096 + 512*160 u64, zeroed) receiving globaltimer stamps of every grid
   barrier of the next sb_draft_loop launches (NULL = off). */
int sb_debug_draft_trace(void* buf);
/* Enable sb_draft_loop (default 0: the per-step forwards measured faster); 0 = it returns SB_EUNSUPPORTED and
   the caller issues per-step forwards. */
int sb_set_draft_loop(int32_t enabled);

/* Compaction (K5): copy KV slabs src_slot[i] -> dst_slot[i] for positions [0, len[i]). */
int sb_kv_compact(const sb_decoder_t* m, const sb_kvcache_t* kv, const int32_t* src_slot,
                  const int32_t* dst_slot, const int32_t* len, int32_t n, void* stream);

/*
 * GEMM entry used by tests/benches: Y[M,N] = X[M,K] W[N,K]^T, fp32 accumulate.
 * epi: 0 store dtype, 1 store fp32, 2 fp32 residual +=, 3 silu(gate)*up on
 * interleaved (gate, up) rows -> [M, N/2].  backend: 0 auto, 1 SIMT (FFMA),
 * 2 tcgen05 (bf16 only; SB_EUNSUPPORTED otherwise), 3 the small-token mma.sync kernel of the draft step
 * (bf16, M <= 16, K = 256 x {1,2,3,4,6,8,12}, epi 0/2/3; SB_EUNSUPPORTED otherwise).  The workspace must be
 * zero-initialised once (stream-K tile counters self-reset).
 */
int sb_gemm(int32_t dtype, const void* x, const void* w, void* y, int32_t M, int32_t N, int32_t K,
            int32_t epi, int32_t backend, void* workspace, size_t ws_bytes, void* stream);
size_t sb_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K);

/* The counter RNG shared with the oracle: u = (mix(seed, stream, ctr) >> 40) * 2^-24. */
float sb_uniform_host(uint64_t seed, uint64_t stream_id, uint64_t counter);

/* One-time host setup (kernel attributes, TMA encoder); call before any graph capture. */
int sb_init(void);
/* Force the forward's GEMM backend (0 auto = tcgen05 for bf16, 1 SIMT, 2 tcgen05); for ablations. */
int sb_set_gemm_backend(int32_t backend);
/* Programmatic dependent launch for every kernel (default on); 0 disables (ablation). */
int sb_set_pdl(int32_t enabled);
/* Diagnostics: skip kernel classes of the bf16 forward (bit 0 attention, 1 qkv, 2 o, 3 gate/up, 4 down) to
   measure their marginal in-graph cost; outputs are meaningless while set.  0 = off. */
int sb_debug_skip(int32_t mask);
/* Diagnostics: per-CTA timeline of the GEMM / attention launches issued after this call (until called
   with NULL; graphs captured meanwhile keep recording).  buf (zeroed, u64): buf[0] = record count, record r
   at buf + 8 + 8r = {launch id, block, smid, t_entry, t_dependency_resolved, t_mainloop_done, t_exit,
   kind (1 gemm, 2 attention)}, globaltimer ns.  The caller sizes buf for the CTAs it launches. */
int sb_debug_cta_trace(void* buf);
/* Experiments: GEMM weight stages requested before the PDL wait (0 = the whole ring) and where the GEMM
   triggers its dependents (0 after its last load, 1 after its epilogue); flags bit 0 skips the epilogue
   stores (outputs meaningless).  Takes effect for later launches. */
int sb_debug_gemm_pdl(int32_t pre_max, int32_t launch_late, int32_t flags);
/* RMSNorm fused into the GEMM epilogues on the bf16 path (default on); 0 = separate norm kernels. */
int sb_set_fuse_norm(int32_t enabled);
/* Decode-sized GEMMs of small models (<= 16 tokens, <= 8M weights: the draft step) on the mma.sync small-token
   kernel (default 1); 0 = every bf16 GEMM on the tcgen05 kernel (A/B, tests). */
int sb_set_small_gemm(int32_t enabled);
/* Diagnostics: eager forward with an event after every kernel; per-stage summed ms as "tag=ms;..." in buf. */
int sb_profile_forward(const sb_decoder_t* m, const sb_kvcache_t* kv, const int32_t* tok_ids,
                       const int32_t* tok_slot, const int32_t* tok_pos, int32_t n_seq, int32_t q_len,
                       float* logits, int32_t logits_mode, void* workspace, size_t ws_bytes, void* stream,
                       char* buf, int32_t buf_len);
/* Attention implementation: 0 tensor-core flash decoding with fused RoPE+append (bf16 default), 1 separate kernels. */
int sb_set_attention_impl(int32_t impl);
/* Flash-decoding key splits of the tensor-core attention: 1 off (default; measured slower), 0 automatic (~2 CTAs per SM), n forced (<= 8). */
int sb_set_attention_splits(int32_t splits);
/* tcgen05 GEMM tuning overrides (0 = automatic): CTAs per SM (1|2), max pipeline stages, K splits. */
int sb_gemm_tune(int32_t ctas_per_sm, int32_t max_stages, int32_t splits);
/*
 * Measure the tcgen05 GEMM configurations (CTAs per SM x K splits) of one
 * shape Y[M,N] = X[M,K] W[N,K]^T on real bf16 operands (y: fp32 [M,N] scratch)
 * and use the fastest for every later GEMM of that (token tile, N, K) shape.
 * Not during graph capture (SB_EINVAL).  Outputs optional.
 */
int sb_gemm_autotune(const void* x, const void* w, void* y_f32, int32_t M, int32_t N, int32_t K, void* stream,
                     int32_t* cps_out, int32_t* splits_out, float* us_out);
int sb_gemm_autotune_clear(void);
/* L2 policy of the weight stream for the next sb_gemm / sb_gemm_autotune calls (0 default, 1 evict-first,
 * 2 evict-last); every decoder forward sets its own (large models evict-first, small ones evict-last). */
int sb_set_weight_l2_hint(int32_t hint);
/*
 * Read / write one entry of the measured table (key: the token tile of M, N, K)
 * so a tuned table can be saved and replayed -- e.g. into a profiler run,
 * whose serialised timings would tune differently.  get: SB_EINVAL if absent.
 */
int sb_gemm_tune_get(int32_t M, int32_t N, int32_t K, int32_t* cps, int32_t* splits, int32_t* weight_tiles,
                     int32_t* token_tile);
int sb_gemm_tune_set(int32_t M, int32_t N, int32_t K, int32_t cps, int32_t splits, int32_t weight_tiles,
                     int32_t token_tile);
int sb_version(void);
const char* sb_build_info(void);
int sb_last_kernel_count(void); /* kernels launched by the last sb_decoder_forward */

#ifdef __cplusplus
}
#endif
#endif /* SPECBATCH_B200_H */
