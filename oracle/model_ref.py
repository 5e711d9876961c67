"""CPU reference of the draft/target decoders and of speculative decoding with
them -- TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py cpu_baseline).

The reference package has no transformer; BASELINE.json asks for
parity "against the reference CPU implementation on identical random-init
weights".  This module is that CPU implementation, written independently of
the product code: plain PyTorch on the CPU, one sequence at a time, fp32 or
fp64, with an optional bf16-rounding emulation that rounds exactly where the
GPU numerics contract (paper_2310_18813_b200/csrc/layer_kernels.cu header)
rounds.  Speculative decoding follows the reference semantics:
LCP verify (engine.py:74-86), advance = min(l+1, remaining) (engine.py:167),
formed batch held until all finish (engine.py:186-188), s=0 plain decoding
(engine.py:158-160).

Parity status: the reference pins only integer semantics; logits parity is
"unpinned by the reference" and is anchored here on (i) the
closed-form identity spec-greedy == plain greedy, and (ii) this oracle.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import spec_ref


def rope_tables(max_pos: int, head_dim: int, theta: float = 10000.0):
    half = head_dim // 2
    inv = theta ** (-(np.arange(half, dtype=np.float64) * 2.0) / head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return torch.from_numpy(np.cos(ang).astype(np.float32)), torch.from_numpy(np.sin(ang).astype(np.float32))


def init_masters(cfg, seed: int, std: float = 0.02, round_to=torch.bfloat16, gain_std: float = 0.1):
    """Independent regeneration of the seeded host init (same draw order as the
    engine's Decoder(init="host")): embed, per layer q,k,v,o,gate,up,down,
    lm_head, then the RMSNorm gains 1 + N(0, gain_std): per layer attn ("ga")
    and mlp ("gm"), then final ("gf")."""
    gen = torch.Generator(device="cpu").manual_seed(seed)
    rn = lambda *shape: torch.randn(*shape, generator=gen, dtype=torch.float32) * std
    h = cfg.hidden
    hd = h // cfg.n_heads
    qd, kd = cfg.n_heads * hd, cfg.n_kv_heads * hd
    r = (lambda t: t.to(round_to).float()) if round_to is not None else (lambda t: t)
    out = {"embed": r(rn(cfg.vocab, h)), "layers": []}
    for _ in range(cfg.n_layers):
        lay = {"wq": rn(qd, h), "wk": rn(kd, h), "wv": rn(kd, h), "wo": rn(h, qd), "wg": rn(cfg.ffn, h),
               "wu": rn(cfg.ffn, h), "wd": rn(h, cfg.ffn)}
        out["layers"].append({k: r(v) for k, v in lay.items()})
    out["lm_head"] = r(rn(cfg.vocab, h))
    gain = lambda: 1.0 + torch.randn(h, generator=gen, dtype=torch.float32) * gain_std
    for lay in out["layers"]:
        lay["ga"] = r(gain())
        lay["gm"] = r(gain())
    out["gf"] = r(gain())
    return out


class LlamaRef:
    """Llama-style decoder on the CPU with a per-sequence KV cache.

    dtype: torch.float32 or torch.float64 compute.  bf16_emulation rounds
    to bf16 where the GPU rounds (GEMM inputs, qkv, rotated q/k, attention
    output, silu*up); the residual stream stays in `dtype`.  RMSNorm is
    y = x * rsqrt(mean(x^2) + eps) * g with per-layer gains g (masters keys
    "ga" before q/k/v, "gm" before gate/up, "gf" before the lm_head; ones
    when absent).  With bf16_emulation it follows the GPU's fused contract:
    the GEMM input is bf16(x * g) and 1/rms scales the GEMM output; in
    fp32/fp64 the two orders are the same math.
    """

    def __init__(self, masters: dict, n_heads: int, n_kv_heads: int, eps: float, max_pos: int = 4096,
                 theta: float = 10000.0, dtype=torch.float64, bf16_emulation: bool = False, n_layers=None,
                 head_dim=None, tp_reduce=None, tp_gather=None):
        """head_dim / tp_reduce / tp_gather describe a tensor-parallel SHARD
        (local head counts, sliced masters): tp_reduce sums the row-parallel
        o / down partials over ranks, tp_gather concatenates the vocab slices."""
        self.dt = dtype
        self.emb = masters["embed"].to(dtype)
        self.head = masters["lm_head"].to(dtype)
        lays = masters["layers"] if n_layers is None else masters["layers"][:n_layers]
        self.layers = [{k: v.to(dtype) for k, v in lay.items()} for lay in lays]
        self.h = self.emb.shape[1]
        one = torch.ones(self.h, dtype=dtype)
        for lay in self.layers:
            lay.setdefault("ga", one)
            lay.setdefault("gm", one)
        self.gf = masters["gf"].to(dtype) if "gf" in masters else one
        self.nq, self.nkv = n_heads, n_kv_heads
        self.hd = head_dim or self.h // n_heads
        self.tp_reduce = tp_reduce or (lambda t: t)
        self.tp_gather = tp_gather or (lambda t: t)
        self.eps = eps
        cos, sin = rope_tables(max_pos, self.hd, theta)
        self.cos, self.sin = cos.to(dtype), sin.to(dtype)
        self.bf16 = bf16_emulation

    def _r(self, x):
        return x.to(torch.bfloat16).to(self.dt) if self.bf16 else x

    def _norm(self, x, g):
        ms = (x.float() * x.float()).mean(-1, keepdim=True) if self.dt == torch.float32 else (x * x).mean(-1, keepdim=True)
        return self._r(x * torch.rsqrt(ms.to(self.dt) + self.eps) * g)

    def _nm(self, x, W, g):
        """(rmsnorm(x) * g) @ W^T under the numerics contract."""
        if self.bf16:
            inv = torch.rsqrt((x * x).mean(-1, keepdim=True) + self.eps)
            return (self._r(x * g) @ W.T) * inv
        return self._norm(x, g) @ W.T

    def _rope(self, x, pos):  # x [T, heads, hd]
        half = self.hd // 2
        c = self.cos[pos][:, None, :]
        s = self.sin[pos][:, None, :]
        a, b = x[..., :half], x[..., half:]
        return self._r(torch.cat([a * c - b * s, b * c + a * s], -1))

    def new_cache(self):
        return [{"k": None, "v": None} for _ in self.layers]

    @torch.no_grad()
    def forward(self, ids, pos, cache):
        """ids/pos: lists (one sequence, positions contiguous and >= cache length
        of valid entries).  The cache keeps keys by absolute position; entries
        at positions >= pos[0] are overwritten (in-place rollback)."""
        ids_t = torch.as_tensor(ids, dtype=torch.long)
        pos_t = torch.as_tensor(pos, dtype=torch.long)
        x = self.emb[ids_t].clone()
        T = len(ids)
        scale = 1.0 / math.sqrt(self.hd)
        p0 = int(pos[0])
        for lay, c in zip(self.layers, cache):
            q = self._r(self._nm(x, lay["wq"], lay["ga"])).view(T, self.nq, self.hd)
            kk = self._r(self._nm(x, lay["wk"], lay["ga"])).view(T, self.nkv, self.hd)
            vv = self._r(self._nm(x, lay["wv"], lay["ga"])).view(T, self.nkv, self.hd)
            q = self._rope(q, pos_t)
            kk = self._rope(kk, pos_t)
            keep_k = c["k"][:p0] if c["k"] is not None else kk[:0]
            keep_v = c["v"][:p0] if c["v"] is not None else vv[:0]
            c["k"] = torch.cat([keep_k, kk], 0)
            c["v"] = torch.cat([keep_v, vv], 0)
            K, Vv = c["k"], c["v"]
            rep = self.nq // self.nkv
            Kh = K.repeat_interleave(rep, dim=1)  # [S, nq, hd]
            Vh = Vv.repeat_interleave(rep, dim=1)
            qs = q * scale
            att = torch.einsum("tnd,snd->nts", qs, Kh)
            S = K.shape[0]
            mask = torch.arange(S)[None, :] > pos_t[:, None]
            att = att.masked_fill(mask[None], float("-inf"))
            att = torch.softmax(att, -1)
            o = self._r(torch.einsum("nts,snd->tnd", att, Vh).reshape(T, self.nq * self.hd))
            x = x + self.tp_reduce(o @ lay["wo"].T)
            g = self._nm(x, lay["wg"], lay["gm"])
            u = self._nm(x, lay["wu"], lay["gm"])
            a = self._r(torch.nn.functional.silu(g) * u)
            x = x + self.tp_reduce(a @ lay["wd"].T)
        return self.tp_gather(self._nm(x, self.head, self.gf)).to(torch.float64).numpy()


def init_opt_masters(cfg, seed: int, max_pos: int, std: float = 0.02, round_to=torch.bfloat16):
    """Independent regeneration of the engine's OPT host init (decoder.py
    Decoder._init_opt draw order)."""
    gen = torch.Generator(device="cpu").manual_seed(seed)
    rn = lambda *shape: torch.randn(*shape, generator=gen, dtype=torch.float32) * std
    r = (lambda t: t.to(round_to).float()) if round_to is not None else (lambda t: t)
    h = cfg.hidden
    hd = h // cfg.n_heads
    qd, kd = cfg.n_heads * hd, cfg.n_kv_heads * hd
    out = {"embed": r(rn(cfg.vocab, h)), "pos": r(rn(max_pos + cfg.pos_offset, h)), "layers": []}
    for _ in range(cfg.n_layers):
        lay = dict(wq=rn(qd, h), wk=rn(kd, h), wv=rn(kd, h), bq=rn(qd), bk=rn(kd), bv=rn(kd), wo=rn(h, qd), bo=rn(h),
                   f1=rn(cfg.ffn, h), b1=rn(cfg.ffn), f2=rn(h, cfg.ffn), b2=rn(h))
        lay.update(g1=1.0 + rn(h), c1=rn(h), g2=1.0 + rn(h), c2=rn(h))
        out["layers"].append({k: r(v) for k, v in lay.items()})
    out["gf"], out["cf"] = r(1.0 + rn(h)), r(rn(h))
    return out


class OptRef:
    """OPT decoder on the CPU (BASELINE config 2), restated from the public
    architecture: pre-LayerNorm blocks, biased q/k/v/o, learned absolute
    positions at row p + pos_offset, fc1 -> ReLU -> fc2, final LayerNorm,
    lm_head tied to the token embedding.  bf16_emulation rounds where the GPU
    rounds: LayerNorm outputs (GEMM inputs), q/k/v after bias, the attention
    output and relu(fc1); residual stream in `dtype`."""

    def __init__(self, masters: dict, n_heads: int, eps: float, pos_offset: int = 2, dtype=torch.float64,
                 bf16_emulation: bool = False):
        self.dt = dtype
        self.m = {k: (v.to(dtype) if torch.is_tensor(v) else v) for k, v in masters.items() if k != "layers"}
        self.layers = [{k: v.to(dtype) for k, v in lay.items()} for lay in masters["layers"]]
        self.h = self.m["embed"].shape[1]
        self.nq = n_heads
        self.hd = self.h // n_heads
        self.eps, self.off, self.bf16 = eps, pos_offset, bf16_emulation

    def _r(self, x):
        return x.to(torch.bfloat16).to(self.dt) if self.bf16 else x

    def _ln(self, x, g, b):
        mu = x.mean(-1, keepdim=True)
        var = ((x - mu) ** 2).mean(-1, keepdim=True)
        return self._r((x - mu) * torch.rsqrt(var + self.eps) * g + b)

    def new_cache(self):
        return [{"k": None, "v": None} for _ in self.layers]

    @torch.no_grad()
    def forward(self, ids, pos, cache):
        ids_t = torch.as_tensor(ids, dtype=torch.long)
        pos_t = torch.as_tensor(pos, dtype=torch.long)
        x = self.m["embed"][ids_t] + self.m["pos"][pos_t + self.off]
        T, p0 = len(ids), int(pos[0])
        for lay, c in zip(self.layers, cache):
            xn = self._ln(x, lay["g1"], lay["c1"])
            q = self._r(xn @ lay["wq"].T + lay["bq"]).view(T, self.nq, self.hd)
            kk = self._r(xn @ lay["wk"].T + lay["bk"]).view(T, self.nq, self.hd)
            vv = self._r(xn @ lay["wv"].T + lay["bv"]).view(T, self.nq, self.hd)
            keep_k = c["k"][:p0] if c["k"] is not None else kk[:0]
            keep_v = c["v"][:p0] if c["v"] is not None else vv[:0]
            c["k"], c["v"] = torch.cat([keep_k, kk], 0), torch.cat([keep_v, vv], 0)
            att = torch.einsum("tnd,snd->nts", q / math.sqrt(self.hd), c["k"])
            mask = torch.arange(c["k"].shape[0])[None, :] > pos_t[:, None]
            att = torch.softmax(att.masked_fill(mask[None], float("-inf")), -1)
            o = self._r(torch.einsum("nts,snd->tnd", att, c["v"]).reshape(T, self.h))
            x = x + (o @ lay["wo"].T + lay["bo"])
            xn = self._ln(x, lay["g2"], lay["c2"])
            a = self._r(torch.relu(xn @ lay["f1"].T + lay["b1"]))
            x = x + (a @ lay["f2"].T + lay["b2"])
        xn = self._ln(x, self.m["gf"], self.m["cf"])
        return (xn @ self.m["embed"].T).to(torch.float64).numpy()

    @torch.no_grad()
    def forward_batch(self, ids, pos, caches):
        """b sequences x q tokens sharing every weight read (CPU-baseline timing);
        same math as forward."""
        b, q = len(ids), len(ids[0])
        flat = torch.as_tensor([t for row in ids for t in row], dtype=torch.long)
        pflat = torch.as_tensor([p for row in pos for p in row], dtype=torch.long)
        pos_t = [torch.as_tensor(p, dtype=torch.long) for p in pos]
        x = self.m["embed"][flat] + self.m["pos"][pflat + self.off]
        for li, lay in enumerate(self.layers):
            xn = self._ln(x, lay["g1"], lay["c1"])
            Q = self._r(xn @ lay["wq"].T + lay["bq"]).view(b, q, self.nq, self.hd)
            K = self._r(xn @ lay["wk"].T + lay["bk"]).view(b, q, self.nq, self.hd)
            Vv = self._r(xn @ lay["wv"].T + lay["bv"]).view(b, q, self.nq, self.hd)
            outs = []
            for s in range(b):
                c = caches[s][li]
                p0 = int(pos[s][0])
                keep_k = c["k"][:p0] if c["k"] is not None else K[s][:0]
                keep_v = c["v"][:p0] if c["v"] is not None else Vv[s][:0]
                c["k"], c["v"] = torch.cat([keep_k, K[s]], 0), torch.cat([keep_v, Vv[s]], 0)
                att = torch.einsum("tnd,snd->nts", Q[s] / math.sqrt(self.hd), c["k"])
                mask = torch.arange(c["k"].shape[0])[None, :] > pos_t[s][:, None]
                att = torch.softmax(att.masked_fill(mask[None], float("-inf")), -1)
                outs.append(torch.einsum("nts,snd->tnd", att, c["v"]).reshape(q, self.h))
            x = x + (self._r(torch.cat(outs, 0)) @ lay["wo"].T + lay["bo"])
            xn = self._ln(x, lay["g2"], lay["c2"])
            x = x + (self._r(torch.relu(xn @ lay["f1"].T + lay["b1"])) @ lay["f2"].T + lay["b2"])
        xn = self._ln(x, self.m["gf"], self.m["cf"])
        return (xn @ self.m["embed"].T).view(b, q, -1).numpy()


def greedy_decode(model: LlamaRef, prompt, n: int):
    """Plain greedy decoding: the ground truth every speculative run must equal
    (greedy_reference, engine.py:224-227).  Returns (tokens, top2 gaps)."""
    cache = model.new_cache()
    P = len(prompt)
    toks = list(int(t) for t in prompt)
    logits = model.forward(toks, list(range(P)), cache)[-1]
    out, gaps = [], []
    for i in range(n):
        srt = np.sort(logits)
        gaps.append(float(srt[-1] - srt[-2]))
        t = int(np.argmax(logits))
        out.append(t)
        if i + 1 < n:
            toks.append(t)
            logits = model.forward([t], [len(toks) - 1], cache)[-1]
    return out, gaps


def _top2_gap(lg) -> float:
    a = np.partition(np.asarray(lg, np.float64), -2)[-2:]
    return float(abs(a[1] - a[0]))


def spec_generate(target: LlamaRef, draft: LlamaRef, prompts, target_lens, k: int, mode: str = "greedy",
                  seed: int = 0, inj_samples=None, margins: list | None = None):
    """Batched speculative decoding on the CPU with the engine's protocol:
    draft step 1 re-feeds the last two committed tokens, verify feeds
    (x_{n-1}, d_1..d_k), KV rolled back by position.  Uniforms / injected
    lengths come from the same counter RNG as the GPU (spec_ref.uniforms).
    Returns (tokens per sequence, accepted-length log [iters][b]).

    ``margins`` (a list) receives, per iteration, the [b] smallest decision
    margin of each sequence: greedy -- the top-2 logit gap of every argmax
    taken (draft steps, target positions 0..l); stochastic -- the relative
    margins of every draft sample, accept test and resample
    (spec_ref.inverse_cdf_margin / accept_margin).  A GPU divergence is a
    rounding tie only where this margin is tiny."""
    b = len(prompts)
    P = len(prompts[0])
    tc = [target.new_cache() for _ in range(b)]
    dc = [draft.new_cache() for _ in range(b)] if draft is not None else None
    toks = [list(map(int, p)) for p in prompts]
    for s in range(b):
        if P >= 2:
            target.forward(toks[s][:P - 1], list(range(P - 1)), tc[s])
            if draft is not None:
                draft.forward(toks[s][:P - 1], list(range(P - 1)), dc[s])
    produced = np.zeros(b, np.int64)
    tl = np.asarray(target_lens)
    log = []
    it = 0
    while np.any(produced < tl):
        u = spec_ref.uniforms(seed, it, b)
        l_inj = spec_ref.injected_lengths(seed, it, b, inj_samples) if mode == "injected" else None
        drafts = np.zeros((b, k), np.int32)
        q = np.zeros((b, k, target.emb.shape[0]), np.float32) if mode == "stochastic" else None
        p = np.zeros((b, k + 1, target.emb.shape[0]), np.float32) if mode == "stochastic" else None
        t_tok = np.zeros((b, k + 1), np.int32)
        mg = np.full(b, np.inf)
        tgap = np.zeros((b, k + 1))
        for s in range(b):
            n = len(toks[s])
            if k > 0:
                lg = draft.forward(toks[s][n - 2:n] if n >= 2 else toks[s][n - 1:n],
                                   [n - 2, n - 1] if n >= 2 else [n - 1], dc[s])[-1]
                for j in range(1, k + 1):
                    if j > 1:
                        lg = draft.forward([int(drafts[s, j - 2])], [n - 1 + j - 1], dc[s])[-1]
                    if mode == "stochastic":
                        qq = spec_ref.softmax_rows(lg.astype(np.float32)[None])[0]
                        q[s, j - 1] = qq
                        drafts[s, j - 1] = spec_ref.inverse_cdf(qq, u[s, j - 1])
                        if margins is not None:
                            mg[s] = min(mg[s], spec_ref.inverse_cdf_margin(qq, u[s, j - 1]))
                    else:
                        drafts[s, j - 1] = int(np.argmax(lg))
                        if margins is not None:
                            mg[s] = min(mg[s], _top2_gap(lg))
            vin = [toks[s][n - 1]] + [int(x) for x in drafts[s]]
            tl_logits = target.forward(vin, list(range(n - 1, n + k)), tc[s])
            if mode == "stochastic":
                p[s] = spec_ref.softmax_rows(tl_logits.astype(np.float32))
            t_tok[s] = np.argmax(tl_logits, -1)
            if margins is not None and mode == "greedy":
                tgap[s] = [_top2_gap(r) for r in tl_logits]
        acc, adv, out = spec_ref.accept_batch(mode, k, drafts, produced, tl, target_tok=t_tok, p=p, q=q,
                                              u_acc=u[:, k:2 * k], u_res=u[:, 2 * k], l_inj=l_inj)
        if margins is not None:
            for s in range(b):
                if mode == "greedy":
                    mg[s] = min(mg[s], float(tgap[s, :acc[s] + 1].min()))
                elif mode == "stochastic":
                    for j in range(min(int(acc[s]) + 1, k)):
                        d = int(drafts[s, j])
                        mg[s] = min(mg[s], spec_ref.accept_margin(u[s, k + j], q[s, j, d], p[s, j, d]))
                    l = int(acc[s])
                    w = np.maximum(p[s, l] - q[s, l], 0) if l < k else p[s, k]
                    mg[s] = min(mg[s], spec_ref.inverse_cdf_margin(w, u[s, 2 * k]))
            margins.append(mg)
        log.append([int(a) if produced[s] < tl[s] else -1 for s, a in enumerate(acc)])
        for s in range(b):
            if adv[s] > 0:
                toks[s].extend(int(t) for t in out[s, :adv[s]])
                produced[s] += adv[s]
        it += 1
    return [t[P:] for t in toks], log


@torch.no_grad()
def forward_batch(model: LlamaRef, ids, pos, caches):
    """Batched CPU forward (CPU-baseline timing): b sequences x q tokens share
    every weight read (one matmul per projection over all b*q rows); attention
    and KV caches stay per sequence.  Same math as LlamaRef.forward."""
    if isinstance(model, OptRef):
        return model.forward_batch(ids, pos, caches)
    b = len(ids)
    q = len(ids[0])
    flat = torch.as_tensor([t for row in ids for t in row], dtype=torch.long)
    pos_t = [torch.as_tensor(p, dtype=torch.long) for p in pos]
    x = model.emb[flat].clone()
    T = b * q
    scale = 1.0 / math.sqrt(model.hd)
    for li, lay in enumerate(model.layers):
        Q = model._r(model._nm(x, lay["wq"], lay["ga"])).view(b, q, model.nq, model.hd)
        K = model._r(model._nm(x, lay["wk"], lay["ga"])).view(b, q, model.nkv, model.hd)
        Vv = model._r(model._nm(x, lay["wv"], lay["ga"])).view(b, q, model.nkv, model.hd)
        outs = []
        for s in range(b):
            c = caches[s][li]
            qs = model._rope(Q[s], pos_t[s])
            ks = model._rope(K[s], pos_t[s])
            p0 = int(pos[s][0])
            keep_k = c["k"][:p0] if c["k"] is not None else ks[:0]
            keep_v = c["v"][:p0] if c["v"] is not None else Vv[s][:0]
            c["k"] = torch.cat([keep_k, ks], 0)
            c["v"] = torch.cat([keep_v, Vv[s]], 0)
            rep = model.nq // model.nkv
            Kh = c["k"].repeat_interleave(rep, dim=1)
            Vh = c["v"].repeat_interleave(rep, dim=1)
            att = torch.einsum("tnd,snd->nts", qs * scale, Kh)
            mask = torch.arange(Kh.shape[0])[None, :] > pos_t[s][:, None]
            att = torch.softmax(att.masked_fill(mask[None], float("-inf")), -1)
            outs.append(torch.einsum("nts,snd->tnd", att, Vh).reshape(q, model.nq * model.hd))
        o = model._r(torch.cat(outs, 0))
        x = x + o @ lay["wo"].T
        a = model._r(torch.nn.functional.silu(model._nm(x, lay["wg"], lay["gm"])) * model._nm(x, lay["wu"], lay["gm"]))
        x = x + a @ lay["wd"].T
    return model._nm(x, model.head, model.gf).view(b, q, -1).numpy()
