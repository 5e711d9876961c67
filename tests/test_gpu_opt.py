"""OPT family (BASELINE config 2) on the GPU against the CPU oracle
(oracle/model_ref.OptRef) on identical seeded weights: logits within 1e-3
(fp32) / 2e-2 (bf16) of the logit scale, fp32 greedy decoding token for token
(tie-aware), and greedy speculative decoding with a self-speculative OPT
draft == plain greedy."""

import numpy as np
import pytest
import torch

from oracle import model_ref
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.engine import SequenceState
from paper_2310_18813_b200.spec_engine import SpecEngine

pytestmark = pytest.mark.gpu
TIE_GAP = 2e-4


def _oracle(dec, bf16):
    m = model_ref.init_opt_masters(dec.cfg, dec.seed, max_pos=dec.max_pos, round_to=dec.tdtype)
    return model_ref.OptRef(m, dec.cfg.n_heads, dec.cfg.rms_eps, bf16_emulation=bf16)


@pytest.mark.parametrize("dtype,tol", [("fp32", 1e-3), ("bf16", 2e-2)])
def test_opt_logits_match_oracle(cuda_dev, dtype, tol):
    dec = Decoder(CONFIGS["tiny-opt"], dtype=dtype, device=cuda_dev, seed=1, init="host", max_pos=128)
    ref = _oracle(dec, dtype == "bf16")
    b, P = 2, 13
    rng = np.random.default_rng(0)
    ids = rng.integers(0, dec.cfg.vocab, size=(b, P)).astype(np.int32)
    kv = dec.new_kv(b, 64)
    ws = torch.zeros(dec.workspace_bytes(b * P), device=cuda_dev, dtype=torch.uint8)
    lg = torch.zeros(b * P, dec.cfg.vocab, device=cuda_dev)
    slots = torch.arange(b, dtype=torch.int32, device=cuda_dev)
    pos = torch.arange(P, dtype=torch.int32, device=cuda_dev).repeat(b)
    dec.forward(kv, torch.as_tensor(ids.reshape(-1), device=cuda_dev), slots, pos, b, P, lg, N.LOGITS_ALL, ws)
    torch.cuda.synchronize()
    got = lg.cpu().numpy().reshape(b, P, -1)
    for s in range(b):
        want = ref.forward(list(ids[s]), list(range(P)), ref.new_cache())
        err = np.abs(got[s] - want).max() / np.abs(want).max()
        assert err < tol, (s, err)


def test_opt_spec_greedy_equals_oracle_greedy(cuda_dev):
    tgt = Decoder(CONFIGS["tiny-opt"], dtype="fp32", device=cuda_dev, seed=2, init="host", max_pos=128)
    drf = Decoder(CONFIGS["tiny-opt"], dtype="fp32", device=cuda_dev, share_from=tgt, share_layers=1, max_pos=128)
    ref = _oracle(tgt, False)
    eng = SpecEngine(tgt, drf, mode="greedy", max_batch=2, max_k=4, prompt_len=8, max_new=16, seed=3)
    for k in (0, 3):
        states = [SequenceState(request_id=i, target_len=16) for i in range(2)]
        eng.generate(states, k)
        for st in states:
            want, gaps = model_ref.greedy_decode(ref, eng.prompt_fn(st.request_id), st.target_len)
            for i, (a, w) in enumerate(zip(st.tokens, want)):
                if a != w:
                    assert gaps[i] < TIE_GAP, (k, st.request_id, i, a, w, gaps[i])
                    break
