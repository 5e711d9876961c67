"""Riding prefill (sb_decoder_forward_mixed): prompts admitted mid-flight are
prefilled inside the next verify forward.  Parity: the window rows' logits and
the prompts' KV equal (bf16 tolerance) those of a plain verify forward plus a
separate prefill forward; continuous batching with riding prompts serves every
request to its length with the streams of plain generation (bf16: allowing
near-tie divergences in a few streams)."""

import numpy as np
import pytest
import torch

from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder, tiny_pair
from paper_2310_18813_b200.engine import SequenceState
from paper_2310_18813_b200.policy import FixedPolicy
from paper_2310_18813_b200.serving import serve_continuous
from paper_2310_18813_b200.spec_engine import SpecEngine
from paper_2310_18813_b200.traffic import Request

pytestmark = pytest.mark.gpu


def _i32(a, dev):
    return torch.as_tensor(np.asarray(a, dtype=np.int32), device=dev)


@pytest.mark.parametrize("n_ride", [1, 3])
def test_mixed_forward_matches_separate_forwards(cuda_dev, n_ride):
    dec = Decoder(CONFIGS["tiny-target"], dtype="bf16", device=cuda_dev, seed=3, init="device", max_pos=512)
    rng = np.random.default_rng(7)
    b, q, hist, plen = 3, 4, 21, 15
    V = dec.cfg.vocab
    ws = torch.zeros(dec.workspace_bytes(b * q + n_ride * plen + 64), device=cuda_dev, dtype=torch.uint8)
    slots = _i32(range(b), cuda_dev)
    pf_slots = _i32(range(b, b + n_ride), cuda_dev)
    kvs = [dec.new_kv(b + n_ride, 128) for _ in range(2)]
    h_ids = _i32(rng.integers(0, V, size=b * hist), cuda_dev)
    h_pos = _i32(np.tile(np.arange(hist), b), cuda_dev)
    for kv in kvs:  # identical history in both caches
        dec.forward(kv, h_ids, slots, h_pos, b, hist, None, N.LOGITS_NONE, ws)
    w_ids = rng.integers(0, V, size=b * q)
    w_pos = np.tile(np.arange(hist, hist + q), b)
    p_ids = rng.integers(0, V, size=n_ride * plen)
    p_pos = np.tile(np.arange(plen), n_ride)
    # (a) mixed: windows + riding prompts in one forward
    lg_mix = torch.zeros(b * q, V, device=cuda_dev)
    rc = dec.forward_mixed(kvs[0], _i32(np.concatenate([w_ids, p_ids]), cuda_dev), slots,
                           _i32(np.concatenate([w_pos, p_pos]), cuda_dev), b, q, n_ride, plen, pf_slots, lg_mix,
                           N.LOGITS_ALL, ws)
    assert rc == 0
    # (b) separate: the verify forward, then the prompts' own prefill forward
    lg_sep = torch.zeros(b * q, V, device=cuda_dev)
    dec.forward(kvs[1], _i32(w_ids, cuda_dev), slots, _i32(w_pos, cuda_dev), b, q, lg_sep, N.LOGITS_ALL, ws)
    dec.forward(kvs[1], _i32(p_ids, cuda_dev), pf_slots, _i32(p_pos, cuda_dev), n_ride, plen, None, N.LOGITS_NONE,
                ws)
    torch.cuda.synchronize()
    a, s = lg_mix.cpu().numpy(), lg_sep.cpu().numpy()
    assert np.abs(a - s).max() / np.abs(s).max() < 2e-2
    assert (a.argmax(-1) == s.argmax(-1)).mean() >= 0.9
    for t in ("k", "v"):
        ka = getattr(kvs[0], t)[:, b:b + n_ride, :, :plen].float()
        kb = getattr(kvs[1], t)[:, b:b + n_ride, :, :plen].float()
        assert (ka - kb).abs().max().item() <= 2e-2 * kb.abs().max().item()
        assert torch.equal(getattr(kvs[0], t)[:, :b, :, :hist + q], getattr(kvs[1], t)[:, :b, :, :hist + q]) or \
            (getattr(kvs[0], t)[:, :b].float() - getattr(kvs[1], t)[:, :b].float()).abs().max().item() < 5e-2


def test_mixed_forward_unsupported_for_fp32(cuda_dev):
    dec = Decoder(CONFIGS["tiny-target"], dtype="fp32", device=cuda_dev, seed=3, init="device", max_pos=128)
    kv = dec.new_kv(2, 64)
    ws = torch.zeros(dec.workspace_bytes(16), device=cuda_dev, dtype=torch.uint8)
    ids = _i32([1, 2, 3, 4, 5], cuda_dev)
    rc = dec.forward_mixed(kv, ids, _i32([0], cuda_dev), _i32([0, 1, 0, 1, 2], cuda_dev), 1, 2, 1, 3,
                           _i32([1], cuda_dev), None, N.LOGITS_NONE, ws)
    assert rc == N.SB_EUNSUPPORTED


def test_continuous_batching_with_riding_prefill(cuda_dev):
    tgt, drf = tiny_pair("bf16", device=cuda_dev, seed=21, max_pos=256)
    eng = SpecEngine(tgt, drf, mode="greedy", max_batch=4, max_k=4, prompt_len=10, max_new=24, seed=5)
    assert eng.supports_ride
    rng = np.random.default_rng(0)
    gens = rng.integers(6, 24, size=12)
    arrivals = np.cumsum(rng.exponential(0.002, size=12))
    wl = [Request(id=i, arrival=float(a), gen_len=int(g)) for i, (a, g) in enumerate(zip(arrivals, gens))]
    rep, extra = serve_continuous(wl, eng, FixedPolicy(3), time_scale=1.0, collect=True, riding=True)
    assert sorted(r.request_id for r in rep.records) == list(range(12))
    assert extra["ridden_rows"] > 0
    same = 0
    for r in wl:
        assert len(extra["outputs"][r.id]) == r.gen_len
        st = SequenceState(request_id=r.id, target_len=r.gen_len)
        eng.generate([st], 0)
        same += extra["outputs"][r.id] == st.tokens
    assert same >= 9, same
