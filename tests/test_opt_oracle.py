"""OPT (config 2) on the CPU: the oracle regenerates the engine's seeded host
init exactly (weights built on the CPU device -- no kernel calls), and the
oracle forward is self-consistent (incremental KV-cache decoding == full
recompute)."""

import numpy as np
import torch

from oracle import model_ref
from paper_2310_18813_b200.decoder import CONFIGS, Decoder


def test_opt_host_init_reproduced():
    cfg = CONFIGS["tiny-opt"]
    dec = Decoder(cfg, dtype="fp32", device="cpu", seed=3, init="host", max_pos=64)
    m = model_ref.init_opt_masters(cfg, 3, max_pos=64, round_to=None)
    assert torch.equal(dec.embed, m["embed"]) and dec.lm_head is dec.embed
    assert torch.equal(dec.pos_embed, m["pos"])
    lay, ref = dec.layers[2], m["layers"][2]
    assert torch.equal(lay["w_qkv"], torch.cat([ref["wq"], ref["wk"], ref["wv"]], 0))
    assert torch.equal(lay["b_qkv"], torch.cat([ref["bq"], ref["bk"], ref["bv"]], 0))
    assert torch.equal(lay["w_gu"], ref["f1"]) and torch.equal(lay["b_fc2"], ref["b2"])
    assert torch.equal(lay["mlp_norm"], ref["g2"]) and torch.equal(lay["attn_norm_b"], ref["c1"])
    assert torch.equal(dec.final_norm_b, m["cf"])
    assert dec.struct.arch == 1 and dec.struct.pos_offset == 2


def test_opt_oracle_incremental_equals_full():
    cfg = CONFIGS["tiny-opt"]
    m = model_ref.init_opt_masters(cfg, 5, max_pos=64, round_to=None)
    ref = model_ref.OptRef(m, cfg.n_heads, cfg.rms_eps)
    ids = list(np.random.default_rng(0).integers(0, cfg.vocab, 12))
    full = ref.forward(ids, list(range(12)), ref.new_cache())
    c = ref.new_cache()
    ref.forward(ids[:8], list(range(8)), c)
    inc = ref.forward(ids[8:], [8, 9, 10, 11], c)
    assert np.abs(full[8:] - inc).max() < 1e-9
