"""The drop-in host API reproduces the REFERENCE package bit-for-bit on the
golden fixtures generated from it (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import paper_2310_18813_b200 as sb
from paper_2310_18813_b200 import cost_model as cm
from paper_2310_18813_b200 import engine as eng
from paper_2310_18813_b200 import policy as pol
from paper_2310_18813_b200 import simulator as sim
from sbtest_util import load_golden


class ConstOracle(eng.DraftOracle):
    def __init__(self, a):
        self.a = a

    def step(self, state, s, rng):
        return min(self.a, s)


def test_tokenlevel_runs_match_reference():
    for case in load_golden("tokenlevel.json"):
        oracle = eng.TokenLevel(case["p_err"], case["seed"])
        states = [eng.SequenceState(rid, tl) for rid, tl in zip(case["request_ids"], case["target_lens"])]
        res = eng.run_batch(states, case["s"], sb.example_calibration(), oracle,
                            np.random.default_rng(case["rng_seed"]))
        assert res.steps == case["result"]["steps"]
        assert res.total_time == case["result"]["total_time"]
        assert res.tokens_generated == case["result"]["tokens_generated"]
        assert {str(k): v for k, v in res.per_sequence_finish.items()} == case["result"]["finish"]
        for st in states:
            assert st.tokens == case["tokens"][str(st.request_id)]
            assert st.tokens == eng.greedy_reference(oracle, st.request_id, st.target_len)


def test_engine_kats():
    g = load_golden("engine.json")
    for c in g["verify"]:
        assert eng.verify(c["draft"], c["target"]) == c["l"]
    for c in g["decode_step"]:
        st = eng.SequenceState(0, c["target_len"])
        o = eng.decode_step(st, c["s"], eng.TokenLevel(p_err=c["p_err"]), np.random.default_rng(1234))
        assert (o.accepted, o.advanced, st.tokens) == (c["accepted"], c["advanced"], c["tokens"])
    simple = sb.LinearStepModel(alpha={1: 1.0}, beta=5.0, ssm_step={1: 0.2})
    for c in g["run_batch_const"]:
        r = eng.run_batch([eng.SequenceState(0, c["n"])], c["s"], simple, ConstOracle(c["a"]),
                          np.random.default_rng(0))
        assert (r.steps, r.total_time) == (c["steps"], c["total_time"])
    cal, trace = sb.example_calibration(), sb.example_trace()
    for c in g["trace_sampler"]:
        states = [eng.SequenceState(i, c["n"]) for i in range(c["b"])]
        r = eng.run_batch(states, c["s"], cal, eng.TraceSampler(trace), np.random.default_rng(c["seed"]))
        assert r.steps == c["steps"] and r.total_time == c["total_time"]
        assert {str(k): v for k, v in r.per_sequence_finish.items()} == c["finish"]


def test_policy_matches_reference():
    g = load_golden("policy.json")
    cal, trace, fit = sb.example_calibration(), sb.example_trace(), sb.example_fit()
    norm = lambda d: {str(k): v for k, v in d.items()}
    assert norm(pol.build_lut(cal, trace).entries) == g["analytic_trace"]
    assert norm(pol.build_lut(cal, fit).entries) == g["analytic_fit"]
    lut = pol.build_lut(cal, trace, mode="simulated", sample_size=200, rng=np.random.default_rng(1))
    assert norm(lut.entries) == g["simulated_seed1"]
    lut = pol.build_lut(cal, trace, mode="simulated", sample_size=40, profiled_sizes=(1, 4, 16),
                        rng=np.random.default_rng(7))
    assert norm(lut.entries) == g["simulated_seed7_small"]
    ref_lut = pol.SpeculationLUT(entries={1: 6, 2: 5, 4: 4, 8: 3, 16: 2, 32: 2}, s_grid=tuple(range(9)))
    for b, s, src in g["lookup"]:
        d = pol.lookup(ref_lut, b)
        assert (d.chosen_s, d.source) == (s, src)
    sizes = (1, 2, 4, 8, 16, 32)
    for c in g["random_calibrations"]:
        model = sb.LinearStepModel(alpha=dict(zip(sizes, c["alpha"])), beta=c["beta"],
                                   ssm_step=dict(zip(sizes, c["ssm"])))
        lut = pol.build_lut(model, sb.PowerLawFit(c=c["c"], gamma=c["gamma"]), profiled_sizes=sizes)
        assert norm(lut.entries) == c["lut"]


def test_serving_matches_reference():
    cal, trace = sb.example_calibration(), sb.example_trace()
    lut = pol.build_lut(cal, trace)
    mk = {
        "poisson_fixed2": (lambda r: sb.gen_arrivals(sb.TrafficConfig(0.05, 1.0, 120), r), pol.fixed_policy(2)),
        "poisson_adaptive": (lambda r: sb.gen_arrivals(sb.TrafficConfig(0.05, 1.0, 120), r), pol.AdaptivePolicy(lut)),
        "bursty_none": (lambda r: sb.gen_arrivals(sb.TrafficConfig(0.02, 5.0, 200), r), pol.fixed_policy(0)),
        "phased_adaptive": (lambda r: sb.gen_phased(sb.PhaseSchedule(phases=(
            (5.0, sb.TrafficConfig(0.02, 1.0, 10**6)), (5.0, sb.TrafficConfig(0.2, 1.0, 10**6)))), r),
            pol.AdaptivePolicy(lut)),
    }
    for case in load_golden("serving.json"):
        wl_fn, policy = mk[case["name"]]
        wl = wl_fn(np.random.default_rng(42))
        assert [r.arrival for r in wl] == case["arrivals"]
        rep = sim.run_simulation(wl, sim.ServerConfig(policy=policy, max_batch=16), cal, trace,
                                 np.random.default_rng(3))
        assert rep.avg_latency == case["avg_latency"]
        assert [list(t) for t in rep.timeline] == case["timeline"]
        got = [[r.request_id, r.t_a, r.t_start, r.t_b, r.latency, r.served_batch_size, r.used_s] for r in rep.records]
        assert got == case["records"]
        assert rep.policy == case["policy"]


def test_cost_model_matches_reference():
    g = load_golden("cost_model.json")
    cal, fit = sb.example_calibration(), sb.example_fit()
    for b, s, TL, TS, TT, steps, pt in g["predict"]:
        p = cm.predict_runtime(cal, fit, 128, b, s)
        assert [p.T_L, p.T_S, p.T_total, p.expected_steps, p.per_token] == [TL, TS, TT, steps, pt]
    prm = cm.OptimalityParams(alpha_eff=1.0, beta=5.0, c=0.9, gamma=0.548)
    for s, v in g["delta"]:
        assert cm.eval_delta(prm, s) == v
    assert cm.optimal_speculation_continuous(prm, 1, 8, tol=1e-7) == g["root"]
    for b, s in g["discrete"]:
        assert cm.optimal_speculation_discrete(cal, fit, 128, b, range(9)) == s


def test_fits_match_reference():
    """fit_linear_step_time (cost_model.py:145-170) and fit_power_law over the
    Eq.4 censored means (acceptance.py:72-106) reproduce the reference's values."""
    from paper_2310_18813_b200 import acceptance as acc

    g = load_golden("cost_model.json")
    for b, ys, want in g["fit_linear"]:
        smp = [cm.StepTimeSample(batch_size=b, query_len=s, measured_time=y) for s, y in zip(range(1, 9), ys)]
        assert list(cm.fit_linear_step_time(smp)) == want
    trace = sb.example_trace()
    pts = [(s, acc.estimate_expected_correct(trace, s)) for s in range(1, 9)]
    assert [list(p) for p in pts] == g["power_law"]["points"]
    pl = acc.fit_power_law(pts)
    assert (pl.c, pl.gamma) == (g["power_law"]["c"], g["power_law"]["gamma"])
