"""Tensor-parallel target (BASELINE config 4: Llama-2-70B over 2/4/8 GPUs of
one NVLink box).

Megatron-style sharding of one Llama decoder over `world` ranks, one process
per GPU:

  w_qkv   column-parallel by heads: rank r holds q heads [r*nq/W, (r+1)*nq/W)
          and kv heads [r*nkv/W, ...) -> attention is rank-local (KV cache
          sharded by kv head)
  w_o     row-parallel (its q-head columns)   -> all-reduce of the fp32 partial
  w_gu    column-parallel (ffn rows r*F/W .., gate/up pairs kept interleaved)
  w_down  row-parallel (the same ffn columns) -> all-reduce
  lm_head vocab-parallel (rows r*V/W ..)       -> all-gather of the logits slice
  embed / norms replicated (no collective for the embedding gather)

Two exchange points per layer plus one per forward; everything after the
logits (token selection, accept, commit) runs replicated and bit-identical on
every rank, so the speculative state never needs a collective.  The draft is
replicated (no communication in the draft loop).

Backends of the C-ABI ``sb_collectives_t``:
  NcclTP  -- NCCL over NVLink (production; graph-capturable)
  HostTP  -- torch.distributed (gloo) through ctypes callbacks: lets TP=2 run
             as two processes on ONE GPU for the parity tests (eager only).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import replace

import numpy as np
import torch

from . import _native as N
from .decoder import Decoder, DecoderConfig

__all__ = ["shard_config", "shard_layer", "shard_decoder", "NcclTP", "HostTP"]


def shard_config(cfg: DecoderConfig, world: int) -> DecoderConfig:
    """Local sizes of one rank's shard (head_dim stays the full model's)."""
    if cfg.n_heads % world or cfg.n_kv_heads % world or cfg.ffn % world or cfg.vocab % world:
        raise ValueError(f"{cfg.name}: heads/kv heads/ffn/vocab must divide by world={world}")
    hd = cfg.head_dim
    return _ShardCfg(name=f"{cfg.name}/tp{world}", hidden=cfg.hidden, n_layers=cfg.n_layers,
                     n_heads=cfg.n_heads // world, n_kv_heads=cfg.n_kv_heads // world, ffn=cfg.ffn // world,
                     vocab=cfg.vocab // world, rms_eps=cfg.rms_eps, rope_theta=cfg.rope_theta, hd=hd)


class _ShardCfg(DecoderConfig):
    """DecoderConfig whose head_dim is fixed (hidden / local heads != head_dim)."""

    def __init__(self, hd: int, **kw):
        object.__setattr__(self, "_hd", hd)
        super().__init__(**kw)

    @property
    def head_dim(self) -> int:
        return self._hd


def shard_layer(lay: dict, cfg: DecoderConfig, world: int, rank: int) -> dict:
    """Slice one layer's device weights (layouts of decoder.py) for `rank`."""
    hd, nq, nkv, F = cfg.head_dim, cfg.n_heads, cfg.n_kv_heads, cfg.ffn
    qd, kd = nq * hd, nkv * hd
    q0, q1 = rank * qd // world, (rank + 1) * qd // world
    k0, k1 = rank * kd // world, (rank + 1) * kd // world
    f0, f1 = rank * F // world, (rank + 1) * F // world
    wqkv = lay["w_qkv"]
    return {
        "attn_norm": lay["attn_norm"], "mlp_norm": lay["mlp_norm"],
        "w_qkv": torch.cat([wqkv[q0:q1], wqkv[qd + k0:qd + k1], wqkv[qd + kd + k0:qd + kd + k1]], 0).contiguous(),
        "w_o": lay["w_o"][:, q0:q1].contiguous(),
        "w_gu": lay["w_gu"][2 * f0:2 * f1].contiguous(),  # (gate, up) pairs stay interleaved
        "w_down": lay["w_down"][:, f0:f1].contiguous(),
    }


def shard_decoder(full: Decoder, world: int, rank: int) -> Decoder:
    """A Decoder holding rank `rank`'s shard of `full` (device slices)."""
    cfg = shard_config(full.cfg, world)
    sh = Decoder.__new__(Decoder)
    sh.cfg = cfg
    sh.dtype_name, sh.tdtype, sh.sb_dtype = full.dtype_name, full.tdtype, full.sb_dtype
    sh.device, sh.max_pos, sh.seed = full.device, full.max_pos, full.seed
    v0, v1 = rank * full.cfg.vocab // world, (rank + 1) * full.cfg.vocab // world
    sh.embed, sh.final_norm = full.embed, full.final_norm
    sh.lm_head = full.lm_head[v0:v1].contiguous()
    sh.layers = [shard_layer(lay, full.cfg, world, rank) for lay in full.layers]
    sh.masters = None
    sh.rope_cos, sh.rope_sin = full.rope_cos, full.rope_sin
    sh.world, sh.rank = world, rank
    sh._build_struct()
    return sh


class _TPBase:
    def __init__(self, world: int, rank: int):
        self.world, self.rank = world, rank
        self.struct = N.SbCollectives()

    def attach(self, dec: Decoder) -> None:
        """Make `dec` (a shard) exchange through this group."""
        dec.struct.tp = C.pointer(self.struct)
        dec._tp = self  # keep the callbacks alive as long as the decoder


class NcclTP(_TPBase):
    """NCCL communicator owned by the native library.  `id_bytes` (128) comes
    from rank 0's ``NcclTP.unique_id()``, broadcast by the host."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        N.call("sb_nccl_unique_id", C.cast(buf, C.c_void_p))
        return bytes(buf)

    def __init__(self, world: int, rank: int, id_bytes: bytes):
        super().__init__(world, rank)
        buf = (C.c_uint8 * 128).from_buffer_copy(id_bytes)
        N.call("sb_nccl_collectives_init", C.cast(buf, C.c_void_p), world, rank, C.byref(self.struct))

    def close(self) -> None:
        if self.struct.ctx:
            N.call("sb_nccl_collectives_destroy", C.byref(self.struct))


class HostTP(_TPBase):
    """Exchange through torch.distributed (any backend; gloo in the tests).
    The native forward calls back into Python at each exchange point: the
    stream is synchronised, the device buffer (which must lie inside one of
    the registered workspaces) is reduced / gathered through host memory and
    copied back.  Eager only (not graph-capturable)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        super().__init__(dist.get_world_size(group), dist.get_rank(group))
        self.buffers: list[torch.Tensor] = []
        self._ar = N._ALLREDUCE_FN(self._all_reduce)
        self._ag = N._ALLGATHER_FN(self._all_gather)
        self.struct.all_reduce_sum = self._ar
        self.struct.all_gather = self._ag
        self.struct.world, self.struct.rank = self.world, self.rank
        self.calls = 0

    def register(self, buf: torch.Tensor) -> None:
        self.buffers.append(buf)

    def _view(self, ptr: int, nbytes: int) -> torch.Tensor:
        for b in self.buffers:
            off = ptr - b.data_ptr()
            if 0 <= off and off + nbytes <= b.numel() * b.element_size():
                return b.view(torch.uint8).view(-1)[off:off + nbytes]
        raise RuntimeError("HostTP: exchange buffer outside the registered workspaces")

    @staticmethod
    def _dt(dtype: int):
        return torch.bfloat16 if dtype == N.SB_BF16 else torch.float32

    def _all_reduce(self, ctx, buf, count, dtype, stream) -> int:
        try:
            torch.cuda.synchronize()
            dt = self._dt(dtype)
            v = self._view(buf, count * torch.tensor([], dtype=dt).element_size()).view(dt)
            h = v.float().cpu()
            self.dist.all_reduce(h, group=self.group)
            v.copy_(h.to(dt))
            torch.cuda.synchronize()
            self.calls += 1
            return 0
        except Exception:  # pragma: no cover - surfaced as a native error
            return 1

    def _all_gather(self, ctx, send, recv, count, dtype, stream) -> int:
        try:
            torch.cuda.synchronize()
            dt = self._dt(dtype)
            es = torch.tensor([], dtype=dt).element_size()
            s = self._view(send, count * es).view(dt).cpu()
            parts = [torch.empty_like(s) for _ in range(self.world)]
            self.dist.all_gather(parts, s, group=self.group)
            self._view(recv, self.world * count * es).view(dt).copy_(torch.cat(parts))
            torch.cuda.synchronize()
            self.calls += 1
            return 0
        except Exception:  # pragma: no cover
            return 1
