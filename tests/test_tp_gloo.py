"""world_size-2 gloo test (CPU) of the tensor-parallel decomposition the CUDA
TP path implements (paper_2310_18813_b200/tp.py, csrc/forward.cu): heads /
ffn / vocab sharded, all-reduce after the row-parallel o and down
projections, all-gather of the vocab slices.  Each rank runs the CPU oracle on
its shard and must reproduce the unsharded oracle's logits (fp64)."""

import os
import socket
from dataclasses import replace

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import model_ref
from paper_2310_18813_b200.decoder import CONFIGS


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard_masters(m, cfg, world, rank):
    """The oracle-layout twin of tp.shard_layer (same index ranges)."""
    hd = cfg.hidden // cfg.n_heads
    qd, kd, F, V = cfg.n_heads * hd, cfg.n_kv_heads * hd, cfg.ffn, cfg.vocab
    sl = lambda n: slice(rank * n // world, (rank + 1) * n // world)
    lays = [{"wq": L["wq"][sl(qd)], "wk": L["wk"][sl(kd)], "wv": L["wv"][sl(kd)], "wo": L["wo"][:, sl(qd)],
             "wg": L["wg"][sl(F)], "wu": L["wu"][sl(F)], "wd": L["wd"][:, sl(F)], "ga": L["ga"], "gm": L["gm"]}
            for L in m["layers"]]  # norm gains replicated
    return {"embed": m["embed"], "lm_head": m["lm_head"][sl(V)], "layers": lays, "gf": m["gf"]}


def _worker(rank, world, port, out, kv_heads=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = CONFIGS["tiny-target"]
        if kv_heads is not None:  # GQA: kv_heads / world kv heads per rank (TP=8 on 70B gives 1)
            cfg = replace(cfg, n_kv_heads=kv_heads)
        m = model_ref.init_masters(cfg, 7, round_to=None)
        hd = cfg.hidden // cfg.n_heads

        def reduce(t):
            t = t.contiguous()
            dist.all_reduce(t)
            return t

        def gather(t):
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t.contiguous())
            return torch.cat(parts, -1)

        full = model_ref.LlamaRef(m, cfg.n_heads, cfg.n_kv_heads, cfg.rms_eps, max_pos=64)
        shard = model_ref.LlamaRef(shard_masters(m, cfg, world, rank), cfg.n_heads // world,
                                   cfg.n_kv_heads // world, cfg.rms_eps, max_pos=64, head_dim=hd,
                                   tp_reduce=reduce, tp_gather=gather)
        ids = list(np.random.default_rng(0).integers(0, cfg.vocab, 9))
        a = full.forward(ids, list(range(9)), full.new_cache())
        cache = shard.new_cache()
        b = shard.forward(ids, list(range(9)), cache)
        # a speculative-window-shaped second call against the sharded KV cache
        a2 = full.forward(ids[:3], [9, 10, 11], _prefilled(full, ids))
        b2 = shard.forward(ids[:3], [9, 10, 11], cache)
        # the vocab-parallel greedy reduction (forward.cu tp_lm_head): each rank's local argmax over
        # its vocab slice -> (max, global index) pairs all-gathered -> the max (ties: lowest index)
        # must equal the argmax of the full row
        local = model_ref.LlamaRef(shard_masters(m, cfg, world, rank), cfg.n_heads // world,
                                   cfg.n_kv_heads // world, cfg.rms_eps, max_pos=64, head_dim=hd,
                                   tp_reduce=reduce)  # no gather: this rank's logits slice
        lg = local.forward(ids, list(range(9)), local.new_cache())
        vl = cfg.vocab // world
        pair = torch.tensor(np.stack([lg.max(-1), lg.argmax(-1) + rank * vl], -1), dtype=torch.float64)
        parts = [torch.empty_like(pair) for _ in range(world)]
        dist.all_gather(parts, pair)
        allp = torch.stack(parts)  # [world][rows][2]
        best = [min(range(world), key=lambda w_: (-allp[w_, r, 0].item(), allp[w_, r, 1].item())) for r in range(9)]
        red = [int(allp[best[r], r, 1].item()) for r in range(9)]
        argmax_ok = red == [int(x) for x in a.argmax(-1)]
        out[rank] = (float(np.abs(a - b).max()), float(np.abs(a2 - b2).max()), float(np.abs(a).max()), argmax_ok)
    finally:
        dist.destroy_process_group()


def _prefilled(model, ids):
    c = model.new_cache()
    model.forward(ids, list(range(len(ids))), c)
    return c


import pytest  # noqa: E402


@pytest.mark.parametrize("kv_heads", [None, 2], ids=["mha", "gqa-1kv-per-rank"])
def test_tp_decomposition_two_ranks(kv_heads):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out, kv_heads), nprocs=2, join=True)
    for r in (0, 1):
        e1, e2, scale, argmax_ok = out[r]
        assert e1 < 1e-9 * max(scale, 1.0) and e2 < 1e-9 * max(scale, 1.0), out[r]
        assert argmax_ok, out[r]
