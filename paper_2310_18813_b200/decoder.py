"""Draft / target decoder pair: shapes, seeded random-init weights in the
B200 layout, KV-cache slabs, and the native forward call.

The reference has no neural network (its "draft/target pair" is a
hash-defined toy, ``TokenLevel`` engine.py:121-152); BASELINE.json's configs
name real shapes, so this module builds those shapes with random weights
(there is no network for checkpoints).  Weight layout in HBM, per layer:

  w_qkv  [(nq + 2 nkv) hd, h]   Q | K | V rows          (one TMA stream)
  w_o    [h, nq hd]
  w_gu   [2 ffn, h]             gate/up rows interleaved g0,u0,g1,u1,...
                                (the tcgen05 epilogue pairs adjacent TMEM
                                lanes with one shuffle to emit silu(g)*u)
  w_down [h, ffn]
KV cache: [L][slots][nkv][ctx_max][hd] per K and V (one contiguous slab per
(layer, slot, head) -> the attention kernel streams it linearly).
"""

from __future__ import annotations

import ctypes as C
import json
import os
import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _native as N

__all__ = ["DecoderConfig", "Decoder", "KVCache", "CONFIGS", "rope_table", "tiny_pair"]


@dataclass(frozen=True)
class DecoderConfig:
    name: str
    hidden: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int = 32000
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0
    arch: str = "llama"  # "llama" | "opt" (config 2: LayerNorm+bias, learned positions, ReLU FFN, tied head)
    pos_offset: int = 2  # OPT: position p reads learned row p + 2

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_heads

    @property
    def qkv_rows(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def _per_layer(self) -> int:
        h, qd = self.hidden, self.n_heads * self.head_dim
        if self.arch == "opt":  # qkv, o, fc1, fc2 + their biases + two LayerNorms (gain, bias)
            return h * self.qkv_rows + h * qd + 2 * h * self.ffn + self.qkv_rows + h + self.ffn + h + 4 * h
        return h * self.qkv_rows + h * qd + 3 * h * self.ffn + 2 * h

    def n_params(self, tied: bool = False) -> int:
        h = self.hidden
        tied = tied or self.arch == "opt"
        fin = 2 * h if self.arch == "opt" else h
        return self.vocab * h * (1 if tied else 2) + self.n_layers * self._per_layer() + fin

    def streamed_bytes_per_forward(self, dtype_bytes: int = 2) -> int:
        """Weight bytes one forward streams from HBM (embedding is a gather,
        excluded; lm_head -- tied or not -- and final norm included) -- SURVEY §8(d)."""
        h = self.hidden
        fin = 2 * h if self.arch == "opt" else h
        return (self.n_layers * self._per_layer() + fin + self.vocab * h) * dtype_bytes

    def kv_bytes_per_token(self, dtype_bytes: int = 2) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * dtype_bytes


CONFIGS = {
    # BASELINE config 3 / 5 target and drafts (public model shapes; random init)
    "llama-2-7b": DecoderConfig("llama-2-7b", 4096, 32, 32, 32, 11008, rms_eps=1e-5),
    "llama-68m": DecoderConfig("llama-68m", 768, 2, 12, 12, 3072, rms_eps=1e-6),
    "llama-160m": DecoderConfig("llama-160m", 768, 12, 12, 12, 3072, rms_eps=1e-6),
    "llama-2-70b": DecoderConfig("llama-2-70b", 8192, 80, 64, 8, 28672, rms_eps=1e-5),
    # BASELINE config 1: the small CPU-runnable pair
    "tiny-target": DecoderConfig("tiny-target", 512, 4, 8, 8, 1376, rms_eps=1e-5),
    # BASELINE config 2: OPT-125M draft / OPT-6.7B target (public shapes; random init)
    "opt-125m": DecoderConfig("opt-125m", 768, 12, 12, 12, 3072, vocab=50272, rms_eps=1e-5, arch="opt"),
    "opt-6.7b": DecoderConfig("opt-6.7b", 4096, 32, 32, 32, 16384, vocab=50272, rms_eps=1e-5, arch="opt"),
    "tiny-opt": DecoderConfig("tiny-opt", 512, 4, 8, 8, 2048, vocab=50272, rms_eps=1e-5, arch="opt"),
}


def rope_table(max_pos: int, head_dim: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin [max_pos, head_dim/2] fp32, computed in fp64 on the host so the
    GPU and the CPU oracle rotate with identical constants."""
    half = head_dim // 2
    inv = theta ** (-(np.arange(half, dtype=np.float64) * 2.0) / head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def _randn(shape, gen, device, std):
    return torch.randn(*shape, generator=gen, device=device, dtype=torch.float32) * std


class Decoder:
    """Seeded random-init Llama-style decoder resident on the GPU.

    init="host": fp32 masters drawn on the CPU with ``torch.Generator(seed)`` in
    a fixed order (embed, per layer q,k,v,o,gate,up,down, lm_head, then the
    RMSNorm gains: per layer attn, mlp, then final) -- the CPU oracle
    reproduces them exactly (used by the parity tests).  Gains are
    1 + N(0, gain_std) (non-unit, as in every trained checkpoint; gain_std=0
    gives ones).
    init="device": drawn on the GPU (7B/70B sizes; no CPU copy).
    ``share_from``/``share_layers`` build a self-speculative draft that reuses
    the target's embedding, lm_head and first layers (config 1's pair).
    """

    def __init__(self, cfg: DecoderConfig, dtype: str = "bf16", device="cuda", seed: int = 0,
                 init: str = "host", max_pos: int = 4096, std: float = 0.02, gain_std: float = 0.1,
                 share_from: "Decoder | None" = None, share_layers: int | None = None):
        if dtype not in ("bf16", "fp32"):
            raise ValueError(f"dtype must be bf16 or fp32, got {dtype!r}")
        self.cfg = cfg
        self.dtype_name = dtype
        self.tdtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.sb_dtype = N.SB_BF16 if dtype == "bf16" else N.SB_F32
        self.device = torch.device(device)
        self.max_pos = max_pos
        self.seed = seed
        h, L = cfg.hidden, cfg.n_layers
        if share_from is not None:
            n_share = share_layers if share_layers is not None else L
            base = share_from
            self.embed, self.lm_head, self.final_norm = base.embed, base.lm_head, base.final_norm
            for extra in ("pos_embed", "final_norm_b"):  # OPT
                if hasattr(base, extra):
                    setattr(self, extra, getattr(base, extra))
            self.layers = base.layers[:n_share]
            self.masters = None if base.masters is None else {
                **{k: v for k, v in base.masters.items() if k != "layers"},
                "layers": base.masters["layers"][:n_share],
            }
            self.cfg = replace(cfg, n_layers=n_share, name=f"{base.cfg.name}[:{n_share}]")
        elif cfg.arch == "opt":
            self._init_opt(cfg, init, seed, std, max_pos)
        else:
            gen_dev = "cpu" if init == "host" else self.device
            gen = torch.Generator(device=gen_dev).manual_seed(seed)
            keep = init == "host"
            masters = {"layers": []} if keep else None

            def mk(shape):
                w = _randn(shape, gen, gen_dev, std)
                return w

            emb = mk((cfg.vocab, h))
            if keep:
                masters["embed"] = emb.to(self.tdtype).float()
            self.embed = emb.to(device=self.device, dtype=self.tdtype)
            del emb
            self.layers = []
            qd = cfg.n_heads * cfg.head_dim
            kd = cfg.n_kv_heads * cfg.head_dim
            for _ in range(L):
                wq, wk, wv = mk((qd, h)), mk((kd, h)), mk((kd, h))
                wo = mk((h, qd))
                wg, wu = mk((cfg.ffn, h)), mk((cfg.ffn, h))
                wd = mk((h, cfg.ffn))
                lay = {
                    "w_qkv": torch.cat([wq, wk, wv], 0).to(device=self.device, dtype=self.tdtype),
                    "w_o": wo.to(device=self.device, dtype=self.tdtype),
                    "w_gu": torch.stack([wg, wu], 1).reshape(2 * cfg.ffn, h).to(device=self.device, dtype=self.tdtype),
                    "w_down": wd.to(device=self.device, dtype=self.tdtype),
                }
                if keep:
                    r = lambda t: t.to(self.tdtype).float()
                    masters["layers"].append({"wq": r(wq), "wk": r(wk), "wv": r(wv), "wo": r(wo), "wg": r(wg),
                                              "wu": r(wu), "wd": r(wd)})
                self.layers.append(lay)
                del wq, wk, wv, wo, wg, wu, wd
            head = mk((cfg.vocab, h))
            if keep:
                masters["lm_head"] = head.to(self.tdtype).float()
            self.lm_head = head.to(device=self.device, dtype=self.tdtype)
            del head
            gain = lambda: 1.0 + _randn((h,), gen, gen_dev, gain_std)
            for li, lay in enumerate(self.layers):
                ga, gm = gain(), gain()
                lay["attn_norm"] = ga.to(device=self.device, dtype=self.tdtype)
                lay["mlp_norm"] = gm.to(device=self.device, dtype=self.tdtype)
                if keep:
                    masters["layers"][li].update(ga=ga.to(self.tdtype).float(), gm=gm.to(self.tdtype).float())
            gf = gain()
            self.final_norm = gf.to(device=self.device, dtype=self.tdtype)
            if keep:
                masters["gf"] = gf.to(self.tdtype).float()
            self.masters = masters
        if self.cfg.arch == "opt":  # learned positions: identity rotation tables (cos 1, sin 0)
            cos = np.ones((max_pos, self.cfg.head_dim // 2), np.float32)
            sin = np.zeros_like(cos)
        else:
            cos, sin = rope_table(max_pos, self.cfg.head_dim, self.cfg.rope_theta)
        self.rope_cos = torch.from_numpy(cos).to(self.device)
        self.rope_sin = torch.from_numpy(sin).to(self.device)
        self._build_struct()

    def _init_opt(self, cfg, init, seed, std, max_pos):
        """OPT weights, fp32 masters drawn in a fixed order (oracle/model_ref.py
        init_opt_masters repeats it): embed (= tied lm_head), learned positions
        [max_pos + offset], per layer wq,wk,wv,bq,bk,bv,wo,bo,fc1,b1,fc2,b2,
        ln1 gain/bias, ln2 gain/bias (gains 1 + N(0, std)), final gain/bias."""
        gen_dev = "cpu" if init == "host" else self.device
        gen = torch.Generator(device=gen_dev).manual_seed(seed)
        keep = init == "host"
        h = cfg.hidden
        qd, kd = cfg.n_heads * cfg.head_dim, cfg.n_kv_heads * cfg.head_dim
        mk = lambda *shape: _randn(shape, gen, gen_dev, std)
        dev = lambda t: t.to(device=self.device, dtype=self.tdtype)
        r = lambda t: t.to(self.tdtype).float()
        masters = {"layers": []} if keep else None
        emb, pos = mk(cfg.vocab, h), mk(max_pos + cfg.pos_offset, h)
        self.embed, self.pos_embed = dev(emb), dev(pos)
        self.lm_head = self.embed  # tied
        if keep:
            masters["embed"], masters["pos"] = r(emb), r(pos)
        self.layers = []
        for _ in range(cfg.n_layers):
            wq, wk, wv = mk(qd, h), mk(kd, h), mk(kd, h)
            bq, bk, bv = mk(qd), mk(kd), mk(kd)
            wo, bo = mk(h, qd), mk(h)
            f1, b1, f2, b2 = mk(cfg.ffn, h), mk(cfg.ffn), mk(h, cfg.ffn), mk(h)
            g1, c1, g2, c2 = 1.0 + mk(h), mk(h), 1.0 + mk(h), mk(h)
            self.layers.append({
                "w_qkv": dev(torch.cat([wq, wk, wv], 0)), "b_qkv": dev(torch.cat([bq, bk, bv], 0)),
                "w_o": dev(wo), "b_o": dev(bo), "w_gu": dev(f1), "b_fc1": dev(b1), "w_down": dev(f2), "b_fc2": dev(b2),
                "attn_norm": dev(g1), "attn_norm_b": dev(c1), "mlp_norm": dev(g2), "mlp_norm_b": dev(c2),
            })
            if keep:
                masters["layers"].append({k: r(v) for k, v in dict(
                    wq=wq, wk=wk, wv=wv, bq=bq, bk=bk, bv=bv, wo=wo, bo=bo, f1=f1, b1=b1, f2=f2, b2=b2,
                    g1=g1, c1=c1, g2=g2, c2=c2).items()})
        gf, cf = 1.0 + mk(h), mk(h)
        self.final_norm, self.final_norm_b = dev(gf), dev(cf)
        if keep:
            masters["gf"], masters["cf"] = r(gf), r(cf)
        self.masters = masters

    # ---------------------------------------------------------------- C struct
    def _build_struct(self):
        cfg = self.cfg
        L = cfg.n_layers
        arr = lambda key: (C.c_void_p * L)(*[lay[key].data_ptr() for lay in self.layers])
        self._arrays = {k: arr(k) for k in ("attn_norm", "w_qkv", "w_o", "mlp_norm", "w_gu", "w_down")}
        s = N.SbDecoder()
        s.n_layers, s.hidden, s.n_heads, s.n_kv_heads = L, cfg.hidden, cfg.n_heads, cfg.n_kv_heads
        s.head_dim, s.ffn, s.vocab, s.dtype, s.max_pos = cfg.head_dim, cfg.ffn, cfg.vocab, self.sb_dtype, self.max_pos
        s.rms_eps = cfg.rms_eps
        s.embed, s.final_norm, s.lm_head = self.embed.data_ptr(), self.final_norm.data_ptr(), self.lm_head.data_ptr()
        for k, a in self._arrays.items():
            setattr(s, k, C.cast(a, C.POINTER(C.c_void_p)))
        s.rope_cos, s.rope_sin = self.rope_cos.data_ptr(), self.rope_sin.data_ptr()
        s.arch = N.ARCH_OPT if cfg.arch == "opt" else N.ARCH_LLAMA
        if cfg.arch == "opt":
            for k in ("attn_norm_b", "mlp_norm_b", "b_qkv", "b_o", "b_fc1", "b_fc2"):
                self._arrays[k] = arr(k)
                setattr(s, k, C.cast(self._arrays[k], C.POINTER(C.c_void_p)))
            s.pos_offset, s.pos_embed = cfg.pos_offset, self.pos_embed.data_ptr()
            s.final_norm_b = self.final_norm_b.data_ptr()
            if self.sb_dtype == N.SB_BF16 and self.device.type == "cuda":
                self._build_ln_fusion(s)
        self.struct = s

    def _build_ln_fusion(self, s) -> None:
        """OPT bf16: LayerNorm fused into its consumer GEMMs (csrc/forward.cu forward_opt): for weight W
        behind LayerNorm (gamma, beta), c1 = W gamma and c2 = W beta (fp32, from the bf16 weights the
        kernels use), so W . LN(x) = rstd * W . (x * gamma) - mean * rstd * c1 + c2."""
        L = self.cfg.n_layers

        def wv(w, v):
            return (w.float() @ v.float()).contiguous()

        self._ln = {"qkv_c1": [wv(l["w_qkv"], l["attn_norm"]) for l in self.layers],
                    "qkv_c2": [wv(l["w_qkv"], l["attn_norm_b"]) for l in self.layers],
                    "fc1_c1": [wv(l["w_gu"], l["mlp_norm"]) for l in self.layers],
                    "fc1_c2": [wv(l["w_gu"], l["mlp_norm_b"]) for l in self.layers],
                    "lm_c1": wv(self.lm_head, self.final_norm), "lm_c2": wv(self.lm_head, self.final_norm_b)}
        for k in ("qkv_c1", "qkv_c2", "fc1_c1", "fc1_c2"):
            a = (C.c_void_p * L)(*[t.data_ptr() for t in self._ln[k]])
            self._arrays["ln_" + k] = a
            setattr(s, "ln_" + k, C.cast(a, C.POINTER(C.c_void_p)))
        s.ln_lm_c1, s.ln_lm_c2 = self._ln["lm_c1"].data_ptr(), self._ln["lm_c2"].data_ptr()

    def gemm_shapes(self) -> dict:
        """(N, K, weight tensor) of the GEMMs one forward runs (layer 0 stands for all)."""
        cfg, lay = self.cfg, self.layers[0] if self.layers else None
        H, qd = cfg.hidden, cfg.n_heads * cfg.head_dim
        out = {"lm": (cfg.vocab, H, self.lm_head)}
        if lay is not None:
            gu_n = cfg.ffn if cfg.arch == "opt" else 2 * cfg.ffn
            out.update(qkv=(cfg.qkv_rows, H, lay["w_qkv"]), o=(H, qd, lay["w_o"]), gu=(gu_n, H, lay["w_gu"]),
                       down=(H, cfg.ffn, lay["w_down"]))
        return out

    def autotune(self, token_counts, stream=None, skip=()) -> dict:
        """Measure the tcgen05 GEMM configuration of every projection for the
        token tiles `token_counts` will use (sb_gemm_autotune); later forwards --
        and graphs captured after this -- use the fastest.  bf16 only; returns
        {(name, tokens): (ctas_per_sm, splits, us)}.

        With SB_TUNE_CACHE=<file.json> the table is replayed from the file when
        it covers every shape (no measurement: e.g. under a profiler, whose
        serialised kernels would tune differently) and written there otherwise."""
        if self.sb_dtype != N.SB_BF16 or self.device.type != "cuda":
            return {}
        lib = N.load()
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        shapes = []
        seen = set()
        for T in sorted(set(int(t) for t in token_counts if t > 0)):
            tn = min(256, max(16, (T + 15) // 16 * 16))
            bucket = (tn, (T + tn - 1) // tn)
            if bucket in seen:
                continue
            seen.add(bucket)
            shapes += [(name, T, n, k, w) for name, (n, k, w) in self.gemm_shapes().items() if name not in skip]
        cache = os.environ.get("SB_TUNE_CACHE")
        table = {}
        if cache and os.path.exists(cache):
            with open(cache) as f:
                table = {tuple(e["key"]): e["val"] for e in json.load(f)}
            if all((T, n, k) in table for _, T, n, k, _ in shapes):
                for (T, n, k), (cps, sp, wt, tn) in table.items():
                    N.call("sb_gemm_tune_set", T, n, k, cps, sp, wt, tn)
                return {(name, T): tuple(table[(T, n, k)][:2]) + (None,) for name, T, n, k, _ in shapes}
        res = {}
        # time the plans under the weight-stream L2 policy this model's forwards use (csrc/forward.cu)
        N.call("sb_set_weight_l2_hint", 1 if self.weight_bytes() > (256 << 20) else 2)
        for name, T, n, k, w in shapes:
            x = torch.randn(T, k, device=self.device, dtype=torch.bfloat16)
            y = torch.empty(T, n, device=self.device, dtype=torch.float32)
            cps, sp, us = C.c_int32(), C.c_int32(), C.c_float()
            N.call("sb_gemm_autotune", x.data_ptr(), w.data_ptr(), y.data_ptr(), T, n, k, st, C.byref(cps),
                   C.byref(sp), C.byref(us))
            res[(name, T)] = (cps.value, sp.value, us.value)
            if cache:
                wt, tn_ = C.c_int32(), C.c_int32()
                N.call("sb_gemm_tune_get", T, n, k, C.byref(cps), C.byref(sp), C.byref(wt), C.byref(tn_))
                table[(T, n, k)] = [cps.value, sp.value, wt.value, tn_.value]
        torch.cuda.synchronize(self.device)
        if cache:
            with open(cache, "w") as f:
                json.dump([{"key": list(kk), "val": v} for kk, v in sorted(table.items())], f)
        return res

    @property
    def vocab_full(self) -> int:
        """Full vocabulary (a tensor-parallel shard holds vocab / world lm_head rows)."""
        return self.cfg.vocab * getattr(self, "world", 1)

    @property
    def is_tp(self) -> bool:
        """True for a tensor-parallel shard attached to a collectives group (tp.py)."""
        return bool(self.struct.tp)

    def workspace_bytes(self, n_tokens: int) -> int:
        return int(N.load().sb_decoder_workspace_bytes(C.byref(self.struct), n_tokens))

    def new_kv(self, slots: int, ctx_max: int) -> "KVCache":
        return KVCache(self, slots, ctx_max)

    def forward(self, kv: "KVCache", ids, slots, pos, n_seq: int, q_len: int, logits, logits_mode: int,
                workspace, stream=None):
        """Launch one forward on ``stream`` (default: torch's current stream)."""
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        N.call("sb_decoder_forward", C.byref(self.struct), C.byref(kv.struct), N.ptr(ids), N.ptr(slots),
               N.ptr(pos), n_seq, q_len, N.ptr(logits), logits_mode, N.ptr(workspace), workspace.numel(), st)

    def forward_greedy(self, kv: "KVCache", ids, slots, pos, n_seq: int, q_len: int, logits, logits_mode: int,
                       workspace, sink: "N.SbTokenSink", stream=None):
        """Forward whose lm_head epilogue emits the greedy token of every row into
        ``sink`` (logits may be None on the bf16 / tcgen05 path)."""
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        N.call("sb_decoder_forward_ex", C.byref(self.struct), C.byref(kv.struct), N.ptr(ids), N.ptr(slots),
               N.ptr(pos), n_seq, q_len, N.ptr(logits), logits_mode, C.byref(sink), N.ptr(workspace),
               workspace.numel(), st)

    def forward_mixed(self, kv: "KVCache", ids, slots, pos, n_seq: int, q_len: int, pf_n: int, pf_len: int, pf_slots,
                      logits, logits_mode: int, workspace, sink: "N.SbTokenSink | None" = None, stream=None) -> int:
        """Verify windows (n_seq x q_len tokens) plus pf_n riding prompts of pf_len
        tokens in one forward (sb_decoder_forward_mixed): ``ids`` / ``pos`` hold the
        window tokens followed by the prompt tokens.  Returns 0, or SB_EUNSUPPORTED
        when this decoder has no mixed path (caller prefills separately)."""
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        rc = N.load().sb_decoder_forward_mixed(C.byref(self.struct), C.byref(kv.struct), N.ptr(ids), N.ptr(slots),
                                               N.ptr(pos), n_seq, q_len, pf_n, pf_len, N.ptr(pf_slots), N.ptr(logits),
                                               logits_mode, C.byref(sink) if sink is not None else None,
                                               N.ptr(workspace), workspace.numel(), st)
        if rc not in (0, N.SB_EUNSUPPORTED):
            N.check("sb_decoder_forward_mixed", rc)
        return rc

    def kv_compact(self, kv: "KVCache", src_slots, dst_slots, lengths, stream=None) -> None:
        """K5 compaction (sb_kv_compact): KV positions [0, lengths[i]) of slot
        src_slots[i] -> dst_slots[i] in every layer (int32 device tensors)."""
        n = int(src_slots.numel())
        if n == 0:
            return
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        N.call("sb_kv_compact", C.byref(self.struct), C.byref(kv.struct), N.ptr(src_slots), N.ptr(dst_slots),
               N.ptr(lengths), n, st)

    def weight_bytes(self) -> int:
        return self.cfg.streamed_bytes_per_forward(2 if self.dtype_name == "bf16" else 4)


class KVCache:
    """K/V slabs [L][slots][nkv][ctx_max][hd] in the decoder's dtype."""

    def __init__(self, dec: Decoder, slots: int, ctx_max: int):
        cfg = dec.cfg
        shape = (cfg.n_layers, slots, cfg.n_kv_heads, ctx_max, cfg.head_dim)
        self.k = torch.zeros(shape, device=dec.device, dtype=dec.tdtype)
        self.v = torch.zeros(shape, device=dec.device, dtype=dec.tdtype)
        self.slots, self.ctx_max = slots, ctx_max
        s = N.SbKVCache()
        s.k, s.v, s.slots, s.ctx_max = self.k.data_ptr(), self.v.data_ptr(), slots, ctx_max
        self.struct = s


def tiny_pair(dtype: str = "fp32", device="cuda", seed: int = 0, max_pos: int = 1024, draft_layers: int = 1):
    """Config 1 pair: tiny Llama target (h=512, L=4) and a self-speculative draft
    made of the target's first layer + shared embedding / lm_head."""
    tgt = Decoder(CONFIGS["tiny-target"], dtype=dtype, device=device, seed=seed, init="host", max_pos=max_pos)
    drf = Decoder(CONFIGS["tiny-target"], dtype=dtype, device=device, share_from=tgt, share_layers=draft_layers,
                  max_pos=max_pos)
    return tgt, drf
