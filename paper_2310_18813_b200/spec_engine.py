"""SpecEngine: batched speculative decoding on one B200.

``SpecEngine(target, draft).generate(batch, k)`` is the GPU implementation of
the reference's ``run_batch`` hot loop (engine.py:176-221): every iteration is

  prepare -> draft step 1 (2 tokens/seq) -> draft steps 2..k (1 token/seq)
          -> target verify over b(k+1) tokens -> argmax | softmax
          -> accept (K4) -> commit + in-place KV rollback (K5)

all on one stream and captured into ONE CUDA graph per (b, k, mode); state
(tokens, lengths, iteration counter) lives on the device so graph replays are
self-advancing.  The host only replays graphs and, every few iterations,
reads a 4-byte live count (pinned, async) to stop.  The formed batch is held
until every sequence finishes, finished rows are masked (engine.py:186-188).

Acceptance modes:
  greedy      -- LCP of draft tokens and target argmax (engine.py:74-86)
  stochastic  -- speculative sampling with the engine's counter RNG
  injected    -- real draft + verify work, accepted length drawn on device
                 from an AcceptanceTrace (TraceSampler law, engine.py:109-118);
                 used for throughput runs on random weights, where real
                 acceptance is ~0.  Always labelled.
"""

from __future__ import annotations

import ctypes as C
import gc
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .acceptance import AcceptanceTrace
from .decoder import Decoder, KVCache
from .engine import BatchResult, SequenceState

__all__ = ["SpecEngine", "IterationStats"]

_MODES = {"greedy": N.ACCEPT_GREEDY, "stochastic": N.ACCEPT_STOCHASTIC, "injected": N.ACCEPT_INJECTED}
_NU = 64  # uniforms per sequence slot per iteration


@dataclass
class IterationStats:
    prefill_ms: float = 0.0
    decode_ms: float = 0.0
    iterations: int = 0
    syncs: int = 0
    accepted: np.ndarray | None = None  # [iters, b], -1 after finishing
    finish_iter: np.ndarray | None = None
    kernels_per_iteration: int = 0
    graph: bool = True
    extra: dict = field(default_factory=dict)


class SpecEngine:
    def __init__(self, target: Decoder, draft: Decoder | None, *, mode: str = "greedy",
                 acceptance: AcceptanceTrace | None = None, max_batch: int = 8, max_k: int = 8,
                 prompt_len: int = 128, max_new: int = 128, seed: int = 0, use_graphs: bool = True,
                 prompt_fn=None, prefill_chunk_tokens: int = 4096, autotune: bool = True):
        if mode not in _MODES:
            raise ValueError(f"mode must be one of {sorted(_MODES)}, got {mode!r}")
        if mode == "injected" and acceptance is None:
            raise ValueError("injected mode needs an AcceptanceTrace")
        if draft is not None and draft.vocab_full != target.vocab_full:
            raise ValueError("draft and target must share a vocabulary")
        if draft is not None and draft.sb_dtype != target.sb_dtype:
            raise ValueError("draft and target must share a dtype")
        N.load()
        N.init_device()
        self.target, self.draft = target, draft
        if draft is not None and draft is not target:
            draft.struct.role = 1  # decode-sized draft GEMMs on the small-token kernel (sb_decoder_t.role)
        self.mode = mode
        self.mode_id = _MODES[mode]
        self.acceptance = acceptance
        self.max_batch, self.max_k = max_batch, max_k if draft is not None else 0
        self.prompt_len, self.max_new = prompt_len, max_new
        self.seed = seed
        self.use_graphs = use_graphs
        self.prompt_fn = prompt_fn or self._default_prompt
        self.dev = target.device
        V = target.vocab_full
        self.V = V
        B, K = max_batch, self.max_k
        self.cap = prompt_len + max_new + K + 2
        self.ctx_max = self.cap + 1
        if self.ctx_max > target.max_pos or (draft is not None and self.ctx_max > draft.max_pos):
            raise ValueError("rope table shorter than prompt_len + max_new + k")
        i32 = dict(device=self.dev, dtype=torch.int32)
        f32 = dict(device=self.dev, dtype=torch.float32)
        self.kv_t = target.new_kv(B, self.ctx_max)
        self.kv_d = draft.new_kv(B, self.ctx_max) if draft is not None else None
        self.slots = torch.arange(B, **i32)
        self.tokens = torch.zeros(B, self.cap, **i32)
        self.n_tok = torch.zeros(B, **i32)
        self.produced = torch.zeros(B, **i32)
        self.target_len = torch.zeros(B, **i32)
        self.finish_iter = torch.full((B,), -1, **i32)
        self.iter = torch.zeros(1, **i32)
        self.live = torch.zeros(1, **i32)
        self.d1_ids = torch.zeros(B * 2, **i32)
        self.d1_pos = torch.zeros(B * 2, **i32)
        self.ds_ids = torch.zeros(B, **i32)
        self.ds_pos = torch.zeros(B, **i32)
        self.d_base = torch.zeros(B, **i32)
        self.v_ids = torch.zeros(B * (K + 1), **i32)
        self.v_pos = torch.zeros(B * (K + 1), **i32)
        self.uniforms = torch.zeros(B * _NU, **f32)
        self.l_inj = torch.zeros(B, **i32)
        samples = acceptance.samples if acceptance is not None else (0,)
        self.inj_samples = torch.tensor(list(samples), **i32)
        self.d_logits = torch.zeros(B, V, **f32) if draft is not None else None
        self.q_probs = torch.zeros(max(1, B * K), V, **f32) if (draft is not None and mode == "stochastic") else None
        self.t_logits = torch.zeros(B * (K + 1), V, **f32)
        self.t_tok = torch.zeros(B * (K + 1), **i32)
        self.accepted = torch.zeros(B, **i32)
        self.advanced = torch.zeros(B, **i32)
        self.out_tok = torch.zeros(B * (K + 1), **i32)
        self.log_cap = max_new + 4
        self.acc_log = torch.full((self.log_cap, B), -1, **i32)
        # prefill staging
        self.pf_chunk = max(1, prefill_chunk_tokens // max(1, prompt_len - 1))
        pf_tok = self.pf_chunk * max(1, prompt_len - 1)
        self.pf_ids = torch.zeros(pf_tok, **i32)
        self.pf_pos = torch.zeros(pf_tok, **i32)
        self._pf_pos_pattern = torch.arange(max(1, prompt_len - 1), **i32).repeat(self.pf_chunk)
        self.pf_slots = torch.zeros(max(B, self.pf_chunk), **i32)  # KV slots of rows being prefilled (serving.py)
        # (B(k+1) window tokens + one prefill chunk riding along: serving.serve_continuous)
        ws = max(target.workspace_bytes(B * (K + 1) + pf_tok), target.workspace_bytes(pf_tok))
        # riding prefill (sb_decoder_forward_mixed): the fused-norm llama bf16 path, unsharded
        self.supports_ride = (target.sb_dtype == N.SB_BF16 and target.cfg.arch == "llama" and not target.is_tp
                              and prompt_len > 1)
        self.mix_ids = torch.zeros(B * (K + 1) + pf_tok, **i32)
        self.mix_pos = torch.zeros(B * (K + 1) + pf_tok, **i32)
        if draft is not None:
            ws = max(ws, draft.workspace_bytes(2 * B), draft.workspace_bytes(pf_tok))
        if draft is not None:
            ws = max(ws, int(N.load().sb_draft_loop_workspace_bytes(C.byref(draft.struct))))
        self.workspace = torch.zeros(ws, device=self.dev, dtype=torch.uint8)
        self.dl_sync = torch.zeros(8, device=self.dev, dtype=torch.int64)  # sb_draft_loop barrier words
        # the draft's weights re-laid as swizzled 16-row tiles for the one-launch draft loop (K1)
        self.dl_packed = None
        if draft is not None and mode != "stochastic":
            nb = int(N.load().sb_draft_loop_packed_bytes(C.byref(draft.struct)))
            if nb:
                self.dl_packed = torch.empty(nb, device=self.dev, dtype=torch.uint8)
                N.call("sb_draft_loop_pack", C.byref(draft.struct), N.ptr(self.dl_packed), nb,
                       torch.cuda.current_stream(self.dev).cuda_stream)
        self.live_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self.stream = torch.cuda.Stream(device=self.dev)
        self.graphs: dict[tuple[int, int], torch.cuda.CUDAGraph] = {}
        self._iter_kernels: dict[tuple[int, int], int] = {}
        self.stats = IterationStats()
        self.tuning = {}
        self.autotune = autotune
        if autotune:
            # measured GEMM configurations for every token count the target verify
            # can present (b(k+1) rows, b rows for the lm_head); must precede graph capture
            Ts = {b * (k + 1) for b in range(1, B + 1) for k in range(K + 1)} | set(range(1, 2 * B + 1))
            if prompt_len > 1:  # prefill chunks of nb prompts (measured: qkv 6.4 -> 5.2 ms at T=1016)
                Ts |= {nb * (prompt_len - 1) for nb in range(1, min(B, self.pf_chunk) + 1)}
            self.tuning["target"] = target.autotune(Ts)
            if draft is not None:  # draft decode steps: b tokens (2b in step 1); measured 1-2% over the heuristic
                self.tuning["draft"] = draft.autotune({n for b in range(1, B + 1) for n in (b, 2 * b)})

    # ------------------------------------------------------------- prompts
    def _default_prompt(self, request_id: int) -> np.ndarray:
        rng = np.random.default_rng([self.seed, int(request_id)])
        return rng.integers(0, self.V, size=self.prompt_len, dtype=np.int64).astype(np.int32)

    # ------------------------------------------------------------- one iteration
    def _iteration(self, b: int, k: int, ride: int = 0, draft_sync: bool = False) -> None:
        """One speculative iteration over rows [0, b).  ``ride`` > 0 (eager only):
        rows [b, b + ride) hold freshly admitted prompts whose target prefill rides
        inside this iteration's verify forward (sb_decoder_forward_mixed) and whose
        draft prefill runs alongside; they join the next iteration.

        ``draft_sync`` (k = 0 only): also run the draft over the last two committed
        tokens (KV only).  Draft step 1 of a k > 0 iteration re-feeds just those
        two, so the draft KV must be valid up to n_tok - 3; a k = 0 iteration
        advances every row by one token without the draft, which would leave a
        hole once a caller switches k per iteration (serving.serve_continuous)."""
        st = torch.cuda.current_stream(self.dev).cuda_stream
        lib = N.load()
        q_pf = self.prompt_len - 1
        if ride:
            if q_pf < 1 or ride > self.pf_chunk or b + ride > self.max_batch:
                raise ValueError("riding prompts exceed the prefill chunk / batch capacity")
            self.pf_ids[: ride * q_pf].copy_(self.tokens[b:b + ride, :q_pf].reshape(-1))
            self.pf_pos[: ride * q_pf].copy_(self._pf_pos_pattern[: ride * q_pf])
            if self.draft is not None:
                self.draft.forward(self.kv_d, self.pf_ids, self.slots[b:], self.pf_pos, ride, q_pf, None,
                                   N.LOGITS_NONE, self.workspace, st)
        launches = 3  # prepare, accept, commit (+ softmax in stochastic mode)
        V = self.V
        mode = self.mode_id
        sample = mode == N.ACCEPT_STOCHASTIC
        use_draft = k > 0 and self.draft is not None
        sync_draft = draft_sync and k == 0 and self.draft is not None
        N.call("sb_prepare_iteration", b, k, N.ptr(self.tokens), self.cap, N.ptr(self.n_tok),
               N.ptr(self.d1_ids) if use_draft or sync_draft else None,
               N.ptr(self.d1_pos) if use_draft or sync_draft else None,
               N.ptr(self.v_ids), N.ptr(self.v_pos), N.ptr(self.d_base), self.seed, N.ptr(self.iter),
               N.ptr(self.uniforms), _NU, N.ptr(self.inj_samples), self.inj_samples.numel(),
               N.ptr(self.l_inj), st)
        if sync_draft:
            self.draft.forward(self.kv_d, self.d1_ids, self.slots, self.d1_pos, b, 2, None, N.LOGITS_NONE,
                               self.workspace, st)
            launches += lib.sb_last_kernel_count()
        greedy_draft = not sample
        # the fp32 path selects from materialised logits; bf16 (a tensor-parallel shard included: local
        # argmax in the lm_head epilogue, (max, index) pairs across ranks) never materialises them
        need_logits = self.target.sb_dtype != N.SB_BF16
        draft_done = False
        if use_draft and greedy_draft and self.dl_packed is not None:
            # the whole greedy draft loop in one persistent launch (csrc/draft_loop.cu)
            rc = lib.sb_draft_loop(C.byref(self.draft.struct), C.byref(self.kv_d.struct), N.ptr(self.dl_packed), b, k,
                                   N.ptr(self.d1_ids),
                                   N.ptr(self.d1_pos), N.ptr(self.slots), N.ptr(self.d_base), N.ptr(self.v_ids),
                                   N.ptr(self.ds_ids), N.ptr(self.ds_pos), N.ptr(self.workspace),
                                   self.workspace.numel(), N.ptr(self.dl_sync), st)
            if rc == 0:
                draft_done = True
                launches += lib.sb_last_kernel_count()
            elif rc != N.SB_EUNSUPPORTED:
                N.check("sb_draft_loop", rc)
        if use_draft and not draft_done:
            sel = N.SELECT_SAMPLE if sample else N.SELECT_ARGMAX
            u_base = self.uniforms.data_ptr()
            for j in range(1, k + 1):
                if j == 1:
                    ids, pos, q = self.d1_ids, self.d1_pos, 2
                else:
                    ids, pos, q = self.ds_ids, self.ds_pos, 1
                if greedy_draft:
                    sink = N.SbTokenSink(self.v_ids.data_ptr() + j * 4, k + 1, self.ds_ids.data_ptr(),
                                         self.ds_pos.data_ptr(), self.d_base.data_ptr(), j)
                    self.draft.forward_greedy(self.kv_d, ids, self.slots, pos, b, q,
                                              self.d_logits if need_logits else None, N.LOGITS_LAST,
                                              self.workspace, sink, st)
                    launches += lib.sb_last_kernel_count()
                    continue
                self.draft.forward(self.kv_d, ids, self.slots, pos, b, q, self.d_logits, N.LOGITS_LAST,
                                   self.workspace, st)
                launches += lib.sb_last_kernel_count() + 1
                probs = self.q_probs.data_ptr() + (j - 1) * V * 4
                N.call("sb_select_tokens", N.ptr(self.d_logits), b, V, sel, u_base + (j - 1) * 4, _NU,
                       probs, k * V, self.v_ids.data_ptr() + j * 4, k + 1, N.ptr(self.ds_ids),
                       N.ptr(self.ds_pos), N.ptr(self.d_base), j, st)
        T = b * (k + 1)
        if ride:  # window tokens, then the riding prompts, in one token list
            Tp = ride * q_pf
            self.mix_ids[:T].copy_(self.v_ids[:T])
            self.mix_pos[:T].copy_(self.v_pos[:T])
            self.mix_ids[T:T + Tp].copy_(self.pf_ids[:Tp])
            self.mix_pos[T:T + Tp].copy_(self.pf_pos[:Tp])
            sink = None if sample else N.SbTokenSink(self.t_tok.data_ptr(), 1, None, None, None, 0)
            rc = self.target.forward_mixed(self.kv_t, self.mix_ids, self.slots, self.mix_pos, b, k + 1, ride, q_pf,
                                           self.slots[b:], self.t_logits if (sample or need_logits) else None,
                                           N.LOGITS_ALL, self.workspace, sink, st)
            if rc != 0:
                raise N.NativeError("sb_decoder_forward_mixed", rc, "unsupported configuration")
            if sample:
                N.call("sb_softmax_rows", N.ptr(self.t_logits), T, V, N.ptr(self.t_logits), st)
        elif sample:
            self.target.forward(self.kv_t, self.v_ids, self.slots, self.v_pos, b, k + 1, self.t_logits,
                                N.LOGITS_ALL, self.workspace, st)
            launches += lib.sb_last_kernel_count()
            N.call("sb_softmax_rows", N.ptr(self.t_logits), T, V, N.ptr(self.t_logits), st)
            launches += 1
        else:
            sink = N.SbTokenSink(self.t_tok.data_ptr(), 1, None, None, None, 0)
            self.target.forward_greedy(self.kv_t, self.v_ids, self.slots, self.v_pos, b, k + 1,
                                       self.t_logits if need_logits else None, N.LOGITS_ALL, self.workspace, sink,
                                       st)
            launches += lib.sb_last_kernel_count()
        if not ride and not sync_draft:
            self._iter_kernels[(b, k)] = launches
        u_base = self.uniforms.data_ptr()
        N.call("sb_accept", mode, b, k, V, N.ptr(self.t_tok), N.ptr(self.t_logits),
               N.ptr(self.q_probs) if sample and k > 0 else None, self.v_ids.data_ptr() + 4, k + 1,
               u_base + k * 4, u_base + 2 * k * 4, _NU, N.ptr(self.l_inj), N.ptr(self.produced),
               N.ptr(self.target_len), N.ptr(self.accepted), N.ptr(self.advanced), N.ptr(self.out_tok), st)
        N.call("sb_kv_commit", b, k, N.ptr(self.advanced), N.ptr(self.accepted), N.ptr(self.out_tok),
               N.ptr(self.tokens), self.cap, N.ptr(self.n_tok), N.ptr(self.produced), N.ptr(self.target_len),
               N.ptr(self.finish_iter), N.ptr(self.iter), N.ptr(self.live), N.ptr(self.acc_log), self.log_cap, st)

    def tune_riding(self) -> None:
        """Measure GEMM plans for the token counts of riding-prefill iterations
        (b(k+1) window tokens + n prompts), once; call outside graph capture."""
        if getattr(self, "_ride_tuned", False) or not self.supports_ride or not self.autotune:
            return
        q = self.prompt_len - 1
        B, K = self.max_batch, self.max_k
        Ts = {b * (k + 1) + n * q for b in range(1, B) for k in range(K + 1) for n in range(1, min(B - b, self.pf_chunk) + 1)}
        self.tuning["target_riding"] = self.target.autotune(Ts, skip=("lm",))  # the lm_head sees window rows only
        self._ride_tuned = True

    def kernels_per_iteration(self, b: int, k: int) -> int:
        """Native kernel launches in one (b, k) iteration, as counted while it was
        last issued (forward driver count + one per token-level kernel)."""
        return self._iter_kernels.get((b, k), 0)

    def _graph(self, b: int, k: int, draft_sync: bool = False):
        draft_sync = draft_sync and k == 0 and self.draft is not None
        key = (b, k, "sync") if draft_sync else (b, k)
        g = self.graphs.get(key)
        if g is None:
            g = _capture_graph(lambda: self._iteration(b, k, draft_sync=draft_sync), self.stream)
            self.graphs[key] = g
        return g

    # ------------------------------------------------------------- batch lifecycle
    def _load_batch(self, states: list[SequenceState], prompts) -> None:
        """Stage the formed batch: prompts (a [b, P] int32 tensor -- pinned host
        memory is copied asynchronously -- or array-likes / the prompt_fn) go to
        the device token table; lengths and counters reset."""
        b = len(states)
        P = self.prompt_len
        if torch.is_tensor(prompts):
            if tuple(prompts.shape) != (b, P):
                raise ValueError(f"prompts tensor must be [{b}, {P}], got {tuple(prompts.shape)}")
            self.tokens[:b, :P].copy_(prompts.to(torch.int32), non_blocking=True)
        else:
            toks = np.zeros((b, P), dtype=np.int32)
            for i, st in enumerate(states):
                pr = prompts[i] if prompts is not None else self.prompt_fn(st.request_id)
                pr = np.asarray(pr, dtype=np.int32).reshape(-1)
                if pr.size != P:
                    raise ValueError(f"prompt of request {st.request_id} has {pr.size} tokens, engine expects {P}")
                toks[i] = pr
            self.tokens[:b, :P].copy_(torch.from_numpy(toks))
        self.n_tok[:b].fill_(P)
        self.produced[:b].zero_()
        self.target_len[:b].copy_(torch.tensor([st.target_len for st in states], dtype=torch.int32))
        self.finish_iter.fill_(-1)
        self.iter.zero_()
        self.acc_log.fill_(-1)

    def _prefill(self, b: int) -> None:
        P = self.prompt_len
        if P < 2:
            return
        q = P - 1
        for s0 in range(0, b, self.pf_chunk):
            nb = min(self.pf_chunk, b - s0)
            # prompt ids straight from the device token table (no host round trip)
            self.pf_ids[: nb * q].copy_(self.tokens[s0:s0 + nb, :q].reshape(-1))
            self.pf_pos[: nb * q].copy_(self._pf_pos_pattern[: nb * q])
            slots = self.slots[s0:]
            self.target.forward(self.kv_t, self.pf_ids, slots, self.pf_pos, nb, q, None, N.LOGITS_NONE,
                                self.workspace)
            if self.draft is not None:
                self.draft.forward(self.kv_d, self.pf_ids, slots, self.pf_pos, nb, q, None, N.LOGITS_NONE,
                                   self.workspace)

    def generate(self, states: list[SequenceState], k: int, rng=None, prompts=None) -> BatchResult:
        """Run a formed batch to completion at speculation length k.

        ``total_time`` / ``per_sequence_finish`` are CUDA-event milliseconds of
        the decode phase (prefill excluded, as in the reference's cost model,
        SPEC.md:141; reported in ``self.stats.prefill_ms``).  Each state's
        ``tokens`` receives its generated stream and ``produced`` its length.
        """
        if not states:
            raise ValueError("empty batch")
        for st in states:
            if st.produced != 0:
                raise ValueError(f"sequence {st.request_id} is not fresh (produced={st.produced})")
            if st.target_len > self.max_new:
                raise ValueError(f"target_len {st.target_len} exceeds engine max_new {self.max_new}")
        if k < 0:
            raise ValueError(f"s must be >= 0, got {k}")
        b = len(states)
        if b > self.max_batch:
            raise ValueError(f"batch {b} exceeds engine max_batch {self.max_batch}")
        if k > self.max_k:
            if self.draft is None:
                raise ValueError("speculation needs a draft model (k > 0)")
            raise ValueError(f"k={k} exceeds engine max_k {self.max_k}")
        with torch.cuda.stream(self.stream):
            self._load_batch(states, prompts)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            self._prefill(b)
            e1.record()
            graph = self._graph(b, k) if self.use_graphs else None
            ev = [torch.cuda.Event(enable_timing=True)]
            ev[0].record()
            remaining = max(st.target_len for st in states)
            syncs = 0
            while True:
                n_launch = max(1, math.ceil(remaining / (k + 1)))
                for _ in range(n_launch):
                    if graph is not None:
                        graph.replay()
                    else:
                        self._iteration(b, k)
                    e = torch.cuda.Event(enable_timing=True)
                    e.record()
                    ev.append(e)
                self.live_host.copy_(self.live, non_blocking=True)
                self.stream.synchronize()
                syncs += 1
                if int(self.live_host[0]) == 0:
                    break
                rem = (self.target_len[:b] - self.produced[:b]).max().item()
                remaining = max(1, int(rem))
                if len(ev) > 4 * self.max_new + 8:
                    raise RuntimeError("speculative loop failed to terminate")
            torch.cuda.synchronize(self.dev)
        iters = len(ev) - 1
        fin = self.finish_iter[:b].cpu().numpy()
        toks = self.tokens[:b].cpu().numpy()
        produced = self.produced[:b].cpu().numpy()
        P = self.prompt_len
        finish = {}
        for i, st in enumerate(states):
            st.tokens = [int(t) for t in toks[i, P:P + int(produced[i])]]
            st.produced = int(produced[i])
            fi = int(fin[i])
            finish[st.request_id] = ev[0].elapsed_time(ev[fi]) if fi > 0 else 0.0
        total = ev[0].elapsed_time(ev[-1])
        self.stats = IterationStats(
            prefill_ms=e0.elapsed_time(e1), decode_ms=total, iterations=iters, syncs=syncs,
            accepted=self.acc_log.view(-1)[: min(iters, self.log_cap) * b].view(-1, b).cpu().numpy(), finish_iter=fin,
            kernels_per_iteration=self.kernels_per_iteration(b, k), graph=graph is not None,
        )
        return BatchResult(batch_size=b, spec_len=k, total_time=total, steps=iters,
                           tokens_generated=sum(st.target_len for st in states), per_sequence_finish=finish)

    # reference-compatible per-sequence hook (DraftOracle protocol) ----------
    def step(self, state, s, rng):  # pragma: no cover - batched engine
        raise NotImplementedError("SpecEngine is a batched oracle: use run_batch/generate")


# ---------------------------------------------------------------- timing hooks
def _capture_graph(fn, stream) -> "torch.cuda.CUDAGraph":
    """Capture ``fn`` on ``stream`` with the cyclic GC off: a collection inside
    the capture can finalise an older engine (pinned buffers, graphs) whose CUDA
    frees are illegal while a stream captures -- the capture is invalidated."""
    g = torch.cuda.CUDAGraph()
    gc.collect()
    gc_was = gc.isenabled()
    gc.disable()
    try:
        with torch.cuda.stream(stream):
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=stream):
                fn()
    finally:
        if gc_was:
            gc.enable()
    return g


def _timed_graph(fn, reps: int, stream) -> float:
    """Capture ``fn`` once into a CUDA graph, replay it ``reps`` times and return
    the mean CUDA-event milliseconds per replay (after one warm replay)."""
    g = _capture_graph(fn, stream)
    with torch.cuda.stream(stream):
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        e1.synchronize()
    return e0.elapsed_time(e1) / reps


def _stage_context(eng: "SpecEngine", b: int, k: int, ctx: int) -> None:
    """Put b slots at context length ctx with random committed tokens (the KV
    rows are whatever the cache holds: timing only)."""
    if not 2 <= ctx <= eng.cap - k - 1:
        raise ValueError(f"context {ctx} outside the engine's token capacity {eng.cap} (k={k})")
    rng = np.random.default_rng(ctx)
    eng.tokens[:b].copy_(torch.from_numpy(rng.integers(0, eng.V, size=(b, eng.cap)).astype(np.int32)))
    eng.n_tok[:b].fill_(ctx)
    eng.iter.zero_()
    st = torch.cuda.current_stream(eng.dev).cuda_stream
    N.call("sb_prepare_iteration", b, k, N.ptr(eng.tokens), eng.cap, N.ptr(eng.n_tok), N.ptr(eng.d1_ids),
           N.ptr(eng.d1_pos), N.ptr(eng.v_ids), N.ptr(eng.v_pos), N.ptr(eng.d_base), eng.seed, N.ptr(eng.iter),
           N.ptr(eng.uniforms), _NU, None, 0, None, st)
    eng.ds_ids[:b].copy_(eng.v_ids.view(-1)[: b * (k + 1): k + 1])
    eng.ds_pos[:b].copy_(eng.d_base[:b] + 1)
    torch.cuda.synchronize(eng.dev)


def time_verify(self, b: int, k: int, ctx: int = 192, reps: int = 20) -> float:
    """Mean ms of ONE target verify forward over b(k+1) tokens at context ctx."""
    _stage_context(self, b, k, ctx)
    fn = lambda: self.target.forward(self.kv_t, self.v_ids, self.slots, self.v_pos, b, k + 1, self.t_logits,
                                     N.LOGITS_ALL, self.workspace)
    return _timed_graph(fn, reps, self.stream)


def time_draft_step(self, b: int, ctx: int = 192, reps: int = 20) -> float:
    """Mean ms of ONE draft decode step (b sequences x 1 token) incl. token selection."""
    if self.draft is None:
        return 0.0
    _stage_context(self, b, 1, ctx)

    sink = N.SbTokenSink(None, 0, self.ds_ids.data_ptr(), None, None, 0)
    need_logits = self.draft.sb_dtype != N.SB_BF16

    def fn():
        st = torch.cuda.current_stream(self.dev).cuda_stream
        self.draft.forward_greedy(self.kv_d, self.ds_ids, self.slots, self.ds_pos, b, 1,
                                  self.d_logits if need_logits else None, N.LOGITS_LAST, self.workspace, sink, st)

    return _timed_graph(fn, reps, self.stream)


SpecEngine.time_verify = time_verify
SpecEngine.time_draft_step = time_draft_step
