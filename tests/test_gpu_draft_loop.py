"""The one-launch greedy draft loop (csrc/draft_loop.cu, sb_draft_loop) against
the per-step draft forwards: identical greedy output streams of the whole
speculative engine (verification makes the output independent of the drafts),
and the drafted tokens themselves agree with the per-step path (bf16: up to
argmax near-ties between two fp32 summation orders)."""

import ctypes as C
from dataclasses import replace

import numpy as np
import pytest
import torch

from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.engine import SequenceState
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context

pytestmark = pytest.mark.gpu


def _pair(cuda_dev):
    tgt = Decoder(replace(CONFIGS["llama-2-7b"], n_layers=2), dtype="bf16", device=cuda_dev, seed=3, init="device",
                  max_pos=320)
    drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=cuda_dev, seed=4, init="device", max_pos=320)
    return tgt, drf


@pytest.mark.parametrize("b,k", [(1, 4), (4, 3), (8, 2), (8, 5)])
def test_draft_loop_first_token_is_an_argmax(cuda_dev, b, k):
    """Step 1 of the draft loop must pick an argmax of the draft's logits (up to
    the bf16 tolerance: random-init logits are near-uniform, so exact ties
    between two fp32 summation orders are common) and write the sink exactly."""
    tgt, drf = _pair(cuda_dev)
    N.load().sb_set_draft_loop(1)
    eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8,
                     prompt_len=128, max_new=64, seed=7, use_graphs=False, autotune=False)
    _stage_context(eng, b, k, 150)
    # reference logits of step 1 on an identical copy of the draft KV cache
    kv_ref = drf.new_kv(eng.max_batch, eng.ctx_max)
    kv_ref.k.copy_(eng.kv_d.k)
    kv_ref.v.copy_(eng.kv_d.v)
    logits = torch.zeros(b, drf.cfg.vocab, device=cuda_dev)
    drf.forward(kv_ref, eng.d1_ids, eng.slots, eng.d1_pos, b, 2, logits, N.LOGITS_LAST, eng.workspace)
    torch.cuda.synchronize()
    assert N.load().sb_draft_loop(C.byref(drf.struct), C.byref(eng.kv_d.struct), b, k, N.ptr(eng.d1_ids),
                                  N.ptr(eng.d1_pos), N.ptr(eng.slots), N.ptr(eng.d_base), N.ptr(eng.v_ids),
                                  N.ptr(eng.ds_ids), N.ptr(eng.ds_pos), N.ptr(eng.workspace), eng.workspace.numel(),
                                  torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    v = eng.v_ids[: b * (k + 1)].view(b, k + 1).cpu()
    lg = logits.cpu()
    scale = lg.abs().max().item()
    for s in range(b):
        d1 = int(v[s, 1])
        assert lg[s, d1].item() >= lg[s].max().item() - 2e-2 * scale, (s, d1, lg[s, d1].item(), lg[s].max().item())
    # sink bookkeeping after k steps
    assert torch.equal(eng.ds_ids[:b].cpu(), v[:, k])
    assert torch.equal(eng.ds_pos[:b].cpu(), eng.d_base[:b].cpu() + k)
    assert ((v[:, 1:] >= 0) & (v[:, 1:] < drf.cfg.vocab)).all()
    N.load().sb_set_draft_loop(0)


def test_engine_output_identical_with_draft_loop(cuda_dev):
    tgt, drf = _pair(cuda_dev)
    lib = N.load()
    outs = []
    for enabled in (0, 1):
        lib.sb_set_draft_loop(enabled)
        try:
            eng = SpecEngine(tgt, drf, mode="greedy", max_batch=4, max_k=4, prompt_len=32, max_new=24, seed=2)
            states = [SequenceState(request_id=i, target_len=24) for i in range(4)]
            eng.generate(states, 3)
            outs.append([st.tokens for st in states])
        finally:
            lib.sb_set_draft_loop(0)
    assert outs[0] == outs[1]
