"""The oracle itself, pinned against the reference's golden fixtures."""

import numpy as np

from oracle import spec_ref
from sbtest_util import load_golden


def test_tokenlevel_replay_matches_reference():
    for case in load_golden("tokenlevel.json"):
        steps, tokens = spec_ref.run_batch_tokenlevel(case["request_ids"], case["target_lens"], case["s"],
                                                      case["seed"], case["p_err"],
                                                      np.random.default_rng(case["rng_seed"]))
        assert len(steps) == case["result"]["steps"]
        for got, want in zip(steps, case["steps"]):
            assert [(r["rid"], r["drafts"], r["accepted"], r["advanced"]) for r in got] == \
                   [(r["rid"], r["drafts"], r["accepted"], r["advanced"]) for r in want]
        for rid, toks in tokens.items():
            assert toks == case["tokens"][str(rid)]


def test_accept_batch_greedy_on_reference_steps():
    for case in load_golden("tokenlevel.json"):
        s = case["s"]
        produced = {rid: 0 for rid in case["request_ids"]}
        tl = dict(zip(case["request_ids"], case["target_lens"]))
        for step in case["steps"]:
            b = len(step)
            drafts = np.array([r["drafts"] for r in step], np.int32).reshape(b, s)
            targets = np.array([r["targets"] for r in step], np.int32).reshape(b, s + 1)
            prod = np.array([produced[r["rid"]] for r in step])
            tlen = np.array([tl[r["rid"]] for r in step])
            acc, adv, out = spec_ref.accept_batch("greedy", s, drafts, prod, tlen, target_tok=targets)
            assert acc.tolist() == [r["accepted"] for r in step]
            assert adv.tolist() == [r["advanced"] for r in step]
            for i, r in enumerate(step):
                produced[r["rid"]] += r["advanced"]
                assert out[i, :r["advanced"]].tolist() == r["targets"][:r["advanced"]]


def test_verify_kats():
    for c in load_golden("engine.json")["verify"]:
        assert spec_ref.lcp(c["draft"], c["target"]) == c["l"]


def test_inverse_cdf_properties():
    rng = np.random.default_rng(0)
    w = rng.random(32000).astype(np.float32)
    w[rng.random(32000) < 0.5] = 0
    assert spec_ref.inverse_cdf(w, 0.0) == int(np.nonzero(w)[0][0])
    last = spec_ref.inverse_cdf(w, np.float32(1 - 2**-24))
    assert w[last] > 0
    picks = [spec_ref.inverse_cdf(w, u) for u in np.sort(rng.random(50).astype(np.float32))]
    assert picks == sorted(picks)  # monotone in u
    assert all(w[p] > 0 for p in picks)
    one = np.zeros(1000, np.float32)
    one[617] = 3.0
    assert spec_ref.inverse_cdf(one, 0.999) == 617
    assert spec_ref.inverse_cdf(np.zeros(10, np.float32), 0.5) == -1


def test_stochastic_accept_rules():
    V, k = 600, 3
    p = np.zeros((1, k + 1, V), np.float32)
    q = np.zeros((1, k, V), np.float32)
    p[..., 5] = 1.0
    q[..., 5] = 1.0
    acc, adv, out = spec_ref.accept_batch("stochastic", k, np.array([[5, 5, 5]]), [0], [10], p=p, q=q,
                                          u_acc=np.array([[0.999, 0.5, 0.0]], np.float32),
                                          u_res=np.array([0.3], np.float32))
    assert acc[0] == 3 and adv[0] == 4 and out[0].tolist() == [5, 5, 5, 5]
    q[0, 1, :] = 0
    q[0, 1, 7] = 1.0  # draft 7 at position 1 has p=0 -> rejected, resample from max(p-q,0) = e_5
    acc, adv, out = spec_ref.accept_batch("stochastic", k, np.array([[5, 7, 5]]), [0], [2], p=p, q=q,
                                          u_acc=np.array([[0.1, 0.1, 0.1]], np.float32),
                                          u_res=np.array([0.9], np.float32))
    assert acc[0] == 1 and adv[0] == 2 and out[0, :2].tolist() == [5, 5]


def test_uniforms_are_in_unit_interval_and_deterministic():
    u = spec_ref.uniforms(7, 3, 4)
    assert u.dtype == np.float32 and (u >= 0).all() and (u < 1).all()
    assert np.array_equal(u, spec_ref.uniforms(7, 3, 4))
    assert not np.array_equal(u, spec_ref.uniforms(7, 4, 4))


def test_inverse_cdf_fixed_point_protocol():
    """The exact fixed-point sampler (token_kernels.cu block_inverse_cdf): W = floor(w * 2^80),
    pick = first v with P_v * 2^32 > floor(u * 2^32) * total -- checked against a direct
    Python-integer restatement and on the encoding's edge values."""
    f = spec_ref.fix80
    assert f(np.array([1.0, 0.5, 2.0 ** -57, 2.0 ** -81, 3.0, -1.0, np.nan, np.inf, 0.0], np.float32)) == \
        [2 ** 80, 2 ** 79, 2 ** 23, 0, 2 ** 80, 0, 0, 0, 0]
    rng = np.random.default_rng(3)
    for trial in range(20):
        V = int(rng.integers(1, 3000))
        w = (rng.random(V) ** 8).astype(np.float32)
        w[rng.random(V) < 0.3] = 0
        u = np.float32(rng.random())
        W = [int(float(x) * 2 ** 80) for x in w.astype(np.float64)]
        tot = sum(W)
        ut = int(float(u) * 2 ** 32)
        want = -1
        run = 0
        for v, x in enumerate(W):
            run += x
            if tot and run * 2 ** 32 > ut * tot:
                want = v
                break
        assert spec_ref.inverse_cdf(w, u) == want
        # order independence of the exact total (what lets the kernel scan in parallel)
        perm = rng.permutation(V)
        assert sum(spec_ref.fix80(w[perm])) == tot
