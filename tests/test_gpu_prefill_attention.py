"""Prefill-sized windows (q_len > 16 / group) run the tensor-core flash
attention in 16-row query blocks after rope_append (attn_tc.cuh block mode).
Parity: the same bf16 forward with the SIMT attention kernel
(sb_set_attention_impl(1)) -- identical GEMMs, fp32 softmax in both -- and,
through test_gpu_model.test_forward_logits_match_oracle (P=21), the fp64 oracle."""

import numpy as np
import pytest
import torch

from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import DecoderConfig, Decoder

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [
    DecoderConfig("mha-hd64", 512, 2, 8, 8, 1024),     # group 1: 16-token blocks
    DecoderConfig("gqa-hd128", 1024, 2, 8, 2, 2048),   # group 4: 4-token blocks
])
@pytest.mark.parametrize("b,q_len", [(3, 37), (1, 127), (2, 17)])
def test_prefill_tc_attention_matches_simt(cuda_dev, cfg, b, q_len):
    dec = Decoder(cfg, dtype="bf16", device=cuda_dev, seed=5, init="device", max_pos=512)
    lib = N.load()
    rng = np.random.default_rng(1)
    T = b * q_len
    ids = torch.as_tensor(rng.integers(0, cfg.vocab, size=T).astype(np.int32), device=cuda_dev)
    # ragged start positions: a prompt continuing after an earlier chunk (history keys already cached)
    start = [0, 40, 7][:b]
    pos = torch.cat([torch.arange(s, s + q_len, dtype=torch.int32) for s in start]).to(cuda_dev)
    slots = torch.arange(b, dtype=torch.int32, device=cuda_dev)
    ws = torch.zeros(dec.workspace_bytes(max(T, 64)), device=cuda_dev, dtype=torch.uint8)
    outs = []
    for impl in (1, 0):
        lib.sb_set_attention_impl(impl)
        try:
            kv = dec.new_kv(b, 256)
            # history for the ragged starts: one plain forward of positions [0, start)
            for s_i, s in enumerate(start):
                if s:
                    hid = torch.as_tensor(rng.integers(0, cfg.vocab, size=s).astype(np.int32), device=cuda_dev)
                    hid_pos = torch.arange(s, dtype=torch.int32, device=cuda_dev)
                    dec.forward(kv, hid, slots[s_i:s_i + 1], hid_pos, 1, s, None, N.LOGITS_NONE, ws)
            rng = np.random.default_rng(1)  # same history tokens for both impls
            rng.integers(0, cfg.vocab, size=T)
            logits = torch.zeros(T, cfg.vocab, device=cuda_dev)
            dec.forward(kv, ids, slots, pos, b, q_len, logits, N.LOGITS_ALL, ws)
            torch.cuda.synchronize()
            outs.append(logits.cpu().numpy())
        finally:
            lib.sb_set_attention_impl(0)
    ref, got = outs
    rel = np.abs(got - ref).max() / np.abs(ref).max()
    assert rel < 2e-2, rel
    # argmax agreement except at near-ties (random-init logits: top-2 gaps within bf16 noise)
    srt = np.sort(ref, axis=-1)
    clear = (srt[:, -1] - srt[:, -2]) > 2e-2 * np.abs(ref).max()
    assert (got.argmax(-1) == ref.argmax(-1))[clear].all()
