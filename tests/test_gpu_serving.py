"""Continuous batching (paper_2310_18813_b200/serving.py): requests admitted
into freed KV slots mid-flight and retired per iteration must produce exactly
the token streams of plain one-batch generation (fp32 greedy: the engine is
batch-invariant, so slot / row / batch-size changes cannot change a stream),
with k re-chosen per iteration by the policy."""

import numpy as np
import pytest
import torch

from oracle import model_ref

from paper_2310_18813_b200.decoder import tiny_pair
from paper_2310_18813_b200.engine import SequenceState
from paper_2310_18813_b200.policy import FixedPolicy, PolicyDecision
from paper_2310_18813_b200.serving import serve_continuous
from paper_2310_18813_b200.spec_engine import SpecEngine
from paper_2310_18813_b200.traffic import Request

pytestmark = pytest.mark.gpu


class _ByBatch:
    """k = 4 for small live batches, 1 for large (exercises per-iteration k switches)."""

    label = "by-batch"

    def decide(self, b):
        return PolicyDecision(b, 4 if b <= 2 else 1, "test")


@pytest.mark.parametrize("policy", [FixedPolicy(3), _ByBatch()], ids=["fixed3", "by-batch"])
def test_continuous_streams_equal_plain_generation(cuda_dev, policy):
    tgt, drf = tiny_pair("fp32", device=cuda_dev, seed=21, max_pos=256)
    eng = SpecEngine(tgt, drf, mode="greedy", max_batch=4, max_k=4, prompt_len=10, max_new=24, seed=5)
    rng = np.random.default_rng(0)
    gens = rng.integers(6, 24, size=11)
    arrivals = np.cumsum(rng.exponential(0.002, size=11))
    wl = [Request(id=i, arrival=float(a), gen_len=int(g)) for i, (a, g) in enumerate(zip(arrivals, gens))]
    rep, extra = serve_continuous(wl, eng, policy, time_scale=1.0, collect=True)
    assert sorted(r.request_id for r in rep.records) == list(range(11))
    assert extra["iterations"] > 0 and extra["mean_live_batch"] <= 4
    for r in wl:  # reference: each request alone through generate()
        st = SequenceState(request_id=r.id, target_len=r.gen_len)
        eng.generate([st], 0)
        assert extra["outputs"][r.id] == st.tokens, r.id
    # and the CPU oracle's plain greedy decoding of every prompt (fp64; tie-aware)
    cfg = tgt.cfg
    ref = model_ref.LlamaRef(tgt.masters, cfg.n_heads, cfg.n_kv_heads, cfg.rms_eps, max_pos=256, dtype=torch.float64)
    ties = 0
    for r in wl:
        want, gaps = model_ref.greedy_decode(ref, eng.prompt_fn(r.id), r.gen_len)
        got = extra["outputs"][r.id]
        d = next((i for i, (a, b_) in enumerate(zip(got, want)) if a != b_), None)
        if d is not None:
            assert gaps[d] < 2e-4, (r.id, d, gaps[d])
            ties += 1
    assert ties <= 1


class _Alternate:
    """k alternates 0, 0, 3 per call: two consecutive k = 0 iterations, then speculation."""

    label = "alternate"

    def __init__(self):
        self.n = 0

    def decide(self, b):
        self.n += 1
        return PolicyDecision(b, 3 if self.n % 3 == 0 else 0, "test")


def test_k0_iterations_keep_draft_kv_current(cuda_dev):
    """a k = 0 iteration advances every row without the draft; draft
    step 1 of the next k > 0 iteration re-feeds only the last two committed
    tokens, so the engine runs the draft over them (KV only) in k = 0
    iterations of serve_continuous.  Draft == target (all 4 layers shared, fp32,
    batch-invariant kernels) must then accept EVERY draft; a stale draft KV
    slot would make the draft's attention read garbage and drop acceptance."""
    tgt, drf = tiny_pair("fp32", device=cuda_dev, seed=23, max_pos=256, draft_layers=4)
    eng = SpecEngine(tgt, drf, mode="greedy", max_batch=4, max_k=4, prompt_len=10, max_new=40, seed=7)
    wl = [Request(id=i, arrival=0.0, gen_len=40) for i in range(3)]
    rep, extra = serve_continuous(wl, eng, _Alternate(), collect=True, riding=False)
    assert extra["acceptance_rate"] == 1.0, extra
    for r in wl:
        st = SequenceState(request_id=r.id, target_len=r.gen_len)
        eng.generate([st], 0)
        assert extra["outputs"][r.id] == st.tokens


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_kv_compact_matches_torch_gather(cuda_dev, dtype):
    """K5 compaction (sb_kv_compact) against a torch copy of the same slab ranges."""
    tgt, _ = tiny_pair(dtype, device=cuda_dev, seed=3, max_pos=256)
    kv = tgt.new_kv(6, 96)
    g = torch.Generator(device=cuda_dev).manual_seed(0)
    kv.k.copy_(torch.randn(kv.k.shape, generator=g, device=cuda_dev).to(kv.k.dtype))
    kv.v.copy_(torch.randn(kv.v.shape, generator=g, device=cuda_dev).to(kv.v.dtype))
    want_k, want_v = kv.k.clone(), kv.v.clone()
    src, dst, lens = [5, 3, 4], [0, 1, 2], [96, 17, 1]
    for s_, d_, n_ in zip(src, dst, lens):
        want_k[:, d_, :, :n_] = want_k[:, s_, :, :n_]
        want_v[:, d_, :, :n_] = want_v[:, s_, :, :n_]
    i32 = dict(device=cuda_dev, dtype=torch.int32)
    tgt.kv_compact(kv, torch.tensor(src, **i32), torch.tensor(dst, **i32), torch.tensor(lens, **i32))
    torch.cuda.synchronize()
    assert torch.equal(kv.k, want_k) and torch.equal(kv.v, want_v)


def test_continuous_with_slot_compaction_equals_plain_generation(cuda_dev):
    """serve_continuous(compact=True): retirements move surviving rows' KV into
    the freed low slots (target and draft caches) so row == slot; the streams
    must stay exactly those of plain generation."""
    tgt, drf = tiny_pair("fp32", device=cuda_dev, seed=21, max_pos=256)
    eng = SpecEngine(tgt, drf, mode="greedy", max_batch=4, max_k=4, prompt_len=10, max_new=24, seed=5)
    rng = np.random.default_rng(1)
    gens = rng.integers(4, 24, size=12)
    arrivals = np.cumsum(rng.exponential(0.002, size=12))
    wl = [Request(id=i, arrival=float(a), gen_len=int(g)) for i, (a, g) in enumerate(zip(arrivals, gens))]
    rep, extra = serve_continuous(wl, eng, _ByBatch(), collect=True, compact=True)
    assert extra["compacted_rows"] > 0, extra
    for r in wl:
        st = SequenceState(request_id=r.id, target_len=r.gen_len)
        eng.generate([st], 0)
        assert extra["outputs"][r.id] == st.tokens, r.id
