"""The persistent single-kernel forward (csrc/persistent.cu) against the
per-layer kernel path on identical weights / inputs: logits within the bf16
tolerance (2e-2 of the logit scale), identical KV-cache appends up to bf16
rounding, fused greedy tokens == argmax of its own logits, and bit-for-bit
determinism across launches.  Shapes: the tiny config-1 target (hd 64), the
LLaMA-68M draft (12 heads of 64) and a 2-layer Llama-2-7B slice (hd 128)."""

from dataclasses import replace

import numpy as np
import pytest
import torch

from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _run(dec, persistent, ids, pos, slots, b, q, logits_mode, ws, kv, sink=None):
    lib = N.load()
    lib.sb_set_persistent(1 if persistent else 0)
    try:
        rows = b if logits_mode == N.LOGITS_LAST else b * q
        logits = torch.zeros(rows, dec.cfg.vocab, device=dec.device)
        if sink is None:
            dec.forward(kv, ids, slots, pos, b, q, logits, logits_mode, ws)
        else:
            dec.forward_greedy(kv, ids, slots, pos, b, q, logits, logits_mode, ws, sink)
        torch.cuda.synchronize()
        return logits
    finally:
        lib.sb_set_persistent(0)


def _case(cfg, cuda_dev, b, P, k, seed=0):
    dec = Decoder(cfg, dtype="bf16", device=cuda_dev, seed=seed, init="device", max_pos=512)
    assert dec.tmaps is not None
    rng = np.random.default_rng(seed)
    slots = torch.arange(b, dtype=torch.int32, device=cuda_dev)
    T = max(b * P, b * (k + 1))
    ws = torch.zeros(dec.workspace_bytes(T), device=cuda_dev, dtype=torch.uint8)
    ids1 = torch.as_tensor(rng.integers(0, cfg.vocab, size=b * P).astype(np.int32), device=cuda_dev)
    pos1 = torch.arange(P, dtype=torch.int32, device=cuda_dev).repeat(b)
    ids2 = torch.as_tensor(rng.integers(0, cfg.vocab, size=b * (k + 1)).astype(np.int32), device=cuda_dev)
    pos2 = (torch.arange(k + 1, dtype=torch.int32, device=cuda_dev) + P).repeat(b)
    return dec, slots, ws, (ids1, pos1), (ids2, pos2)


def _close(a, b):
    scale = max(a.abs().max().item(), 1e-6)
    return (a - b).abs().max().item() / scale


SHAPES = [
    ("tiny", CONFIGS["tiny-target"], 3, 9, 3),
    ("68m", CONFIGS["llama-68m"], 8, 12, 3),
    ("7b-2l", replace(CONFIGS["llama-2-7b"], n_layers=2), 8, 16, 3),
    ("7b-2l-b8k8", replace(CONFIGS["llama-2-7b"], n_layers=2), 8, 20, 8),
    ("7b-1l-long", replace(CONFIGS["llama-2-7b"], n_layers=1), 2, 100, 4),
    ("68m-long", CONFIGS["llama-68m"], 2, 110, 3),
]


@pytest.mark.parametrize("name,cfg,b,P,k", SHAPES, ids=[s[0] for s in SHAPES])
def test_persistent_matches_layered(cuda_dev, name, cfg, b, P, k):
    dec, slots, ws, (ids1, pos1), (ids2, pos2) = _case(cfg, cuda_dev, b, P, k)
    kv_a = dec.new_kv(b, 160)
    kv_b = dec.new_kv(b, 160)
    # prompt (T = b*P) then a speculative window (T = b*(k+1)) on each path
    la1 = _run(dec, False, ids1, pos1, slots, b, P, N.LOGITS_ALL, ws, kv_a)
    lb1 = _run(dec, True, ids1, pos1, slots, b, P, N.LOGITS_ALL, ws, kv_b)
    assert _close(la1, lb1) < TOL, _close(la1, lb1)
    # KV appends agree (bf16 rounding of slightly different fp32 sums)
    ka, kb = kv_a.k.float(), kv_b.k.float()
    assert (ka - kb).abs().max().item() <= TOL * max(ka.abs().max().item(), 1e-6)
    assert (kv_a.v.float() - kv_b.v.float()).abs().max().item() <= TOL * max(kv_a.v.float().abs().max().item(), 1e-6)
    la2 = _run(dec, False, ids2, pos2, slots, b, k + 1, N.LOGITS_ALL, ws, kv_a)
    lb2 = _run(dec, True, ids2, pos2, slots, b, k + 1, N.LOGITS_ALL, ws, kv_b)
    assert _close(la2, lb2) < TOL, _close(la2, lb2)
    # LOGITS_LAST rows == the last row of each sequence
    lb3 = _run(dec, True, ids2, pos2, slots, b, k + 1, N.LOGITS_LAST, ws, kv_b)
    want = lb2.view(b, k + 1, -1)[:, -1]
    assert _close(want, lb3) < 1e-6


def test_persistent_deterministic_and_sink(cuda_dev):
    cfg = replace(CONFIGS["llama-2-7b"], n_layers=2)
    b, P, k = 8, 8, 3
    dec, slots, ws, (ids1, pos1), (ids2, pos2) = _case(cfg, cuda_dev, b, P, k, seed=5)
    kv = dec.new_kv(b, 64)
    _run(dec, True, ids1, pos1, slots, b, P, N.LOGITS_NONE, ws, kv)
    l1 = _run(dec, True, ids2, pos2, slots, b, k + 1, N.LOGITS_ALL, ws, kv)
    l2 = _run(dec, True, ids2, pos2, slots, b, k + 1, N.LOGITS_ALL, ws, kv)
    assert torch.equal(l1, l2)
    T = b * (k + 1)
    out = torch.full((T,), -1, dtype=torch.int32, device=cuda_dev)
    nxt = torch.full((T,), -1, dtype=torch.int32, device=cuda_dev)
    npos = torch.full((T,), -1, dtype=torch.int32, device=cuda_dev)
    base = torch.arange(T, dtype=torch.int32, device=cuda_dev) * 3
    sink = N.SbTokenSink(out.data_ptr(), 1, nxt.data_ptr(), npos.data_ptr(), base.data_ptr(), 7)
    l3 = _run(dec, True, ids2, pos2, slots, b, k + 1, N.LOGITS_ALL, ws, kv, sink=sink)
    assert torch.equal(l1, l3)
    want = torch.argmax(l1, dim=1).to(torch.int32)
    assert torch.equal(out, want) and torch.equal(nxt, want)
    assert torch.equal(npos, base + 7)


def test_persistent_workspace_sync_words_reset(cuda_dev):
    """Back-to-back launches sharing one workspace (draft steps, verify) leave
    the barrier / flag words zero for the next launch."""
    cfg = CONFIGS["llama-68m"]
    b, P, k = 4, 6, 2
    dec, slots, ws, (ids1, pos1), (ids2, pos2) = _case(cfg, cuda_dev, b, P, k, seed=2)
    kv = dec.new_kv(b, 64)
    for _ in range(5):
        _run(dec, True, ids1, pos1, slots, b, P, N.LOGITS_LAST, ws, kv)
    assert int(ws[: 4 * 200].view(torch.int32).abs().sum().item()) == 0


@pytest.mark.parametrize("splits", [2, 4, 8])
def test_attention_key_splits_match_single_pass(cuda_dev, splits):
    """Flash-decoding key splits (sb_set_attention_splits) == one pass over the
    keys: logits within the bf16 tolerance, identical KV appends."""
    lib = N.load()
    cfg = replace(CONFIGS["llama-2-7b"], n_layers=2)
    b, P, k = 2, 150, 3
    dec, slots, ws, (ids1, pos1), (ids2, pos2) = _case(cfg, cuda_dev, b, P, k, seed=9)
    outs = []
    try:
        for sp in (1, splits):
            lib.sb_set_attention_splits(sp)
            kv = dec.new_kv(b, 192)
            _run(dec, False, ids1, pos1, slots, b, P, N.LOGITS_NONE, ws, kv)
            lg = _run(dec, False, ids2, pos2, slots, b, k + 1, N.LOGITS_ALL, ws, kv)
            outs.append((lg, kv.k.clone(), kv.v.clone()))
    finally:
        lib.sb_set_attention_splits(1)
    assert _close(outs[0][0], outs[1][0]) < TOL
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][2], outs[1][2])
