"""The measured profiler and the reference-facing consumers of its output
(SURVEY §8 a10, a12, a13, a15, (f)1): profiler.calibrate on the GPU engine ->
StepTimeSample CSV + calibration JSON in the reference's formats -> the
reference API's build_lut / run_simulation; build_lut(mode="measured") picks
the argmin of its own measured cells; run_simulation(engine=...) serves every
request once through the GPU engine; the accept-kernel log becomes an
AcceptanceTrace."""

import math

import numpy as np
import pytest

from paper_2310_18813_b200 import (AdaptivePolicy, FixedPolicy, ServerConfig, build_lut, example_trace,
                                   run_simulation)
from paper_2310_18813_b200.acceptance import estimate_expected_correct, trace_from_accept_log
from paper_2310_18813_b200.cost_model import (LinearStepModel, llm_step_time, load_calibration, load_step_samples,
                                              save_calibration, save_step_samples)
from paper_2310_18813_b200.decoder import tiny_pair
from paper_2310_18813_b200.engine import SequenceState
from paper_2310_18813_b200.profiler import calibrate
from paper_2310_18813_b200.spec_engine import SpecEngine
from paper_2310_18813_b200.traffic import TrafficConfig, gen_arrivals

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    import torch

    dev = torch.device("cuda:0")
    from paper_2310_18813_b200 import _native

    _native.load()
    _native.init_device()
    tgt, drf = tiny_pair("bf16", device=dev, seed=2, max_pos=256)
    return SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=4, max_k=4, prompt_len=16,
                      max_new=24, seed=3)


def test_calibrate_emits_reference_formats(engine, tmp_path):
    model, samples = calibrate(engine, batch_sizes=(1, 2, 4), k_grid=range(1, 5), reps=3)
    assert isinstance(model, LinearStepModel)
    assert len(samples) == 3 * 4 and all(s.measured_time > 0 for s in samples)
    assert {(s.batch_size, s.query_len) for s in samples} == {(b, s) for b in (1, 2, 4) for s in range(1, 5)}
    a = [model.alpha[b] for b in sorted(model.alpha)]
    assert all(x > 0 for x in a) and a == sorted(a)  # LinearStepModel invariants (cost_model.py:59-85)
    assert all(model.ssm_step[b] > 0 for b in model.ssm_step)
    save_step_samples(samples, tmp_path / "samples.csv")
    back = load_step_samples(tmp_path / "samples.csv")
    assert [(s.batch_size, s.query_len, s.measured_time) for s in back] == \
        [(s.batch_size, s.query_len, s.measured_time) for s in samples]
    save_calibration(model, tmp_path / "cal.json")
    m2, _ = load_calibration(tmp_path / "cal.json")
    assert m2 == model
    # the reference API consumes it unchanged: analytic LUT + virtual-time simulation
    lut = build_lut(m2, example_trace(), s_grid=range(5), profiled_sizes=(1, 2, 4))
    assert set(lut.entries) == {1, 2, 4} and all(0 <= v <= 4 for v in lut.entries.values())
    wl = gen_arrivals(TrafficConfig(0.01, 1.0, 20), np.random.default_rng(0))
    rep = run_simulation(wl, ServerConfig(policy=AdaptivePolicy(lut), max_batch=4), m2, example_trace(),
                         np.random.default_rng(1))
    assert len(rep.records) == 20 and rep.avg_latency > 0
    # the model reproduces its own samples' scale (ms): t_L(b, s) within the sample range per b
    for b in (1, 2, 4):
        ts = [s.measured_time for s in samples if s.batch_size == b]
        assert 0.5 * min(ts) < llm_step_time(m2, b, 2) < 2 * max(ts)


def test_measured_lut_is_argmin_of_its_cells(engine):
    lut = build_lut(None, example_trace(), s_grid=(0, 1, 2, 4), profiled_sizes=(1, 2), mode="measured",
                    sample_size=2, rng=np.random.default_rng(0), gen_len=24, engine=engine)
    cells = lut.provenance["ms_per_token"]
    assert set(cells) == {f"{b},{s}" for b in (1, 2) for s in (0, 1, 2, 4)}
    for b in (1, 2):
        row = {s: cells[f"{b},{s}"] for s in (0, 1, 2, 4)}
        assert all(v > 0 and math.isfinite(v) for v in row.values())
        best = min(row.values())
        assert lut.entries[b] == min(s for s, v in row.items() if v == best)  # ties -> smaller s


def test_run_simulation_on_the_engine(engine):
    wl = gen_arrivals(TrafficConfig(0.002, 1.0, 9), np.random.default_rng(2))
    wl = [type(r)(id=r.id, arrival=r.arrival, gen_len=min(r.gen_len, 24)) for r in wl]
    rep = run_simulation(wl, ServerConfig(policy=FixedPolicy(2), max_batch=4), None, None,
                         np.random.default_rng(0), engine=engine)
    assert sorted(r.request_id for r in rep.records) == list(range(9))
    assert all(r.served_batch_size <= 4 and r.used_s == 2 for r in rep.records)
    assert all(r.t_b > r.t_start >= r.t_a - 1e-12 for r in rep.records)


def test_accept_log_feeds_an_acceptance_trace(engine):
    states = [SequenceState(request_id=i, target_len=24) for i in range(4)]
    engine.generate(states, 4)
    log = engine.stats.accepted
    assert (log < 0).any()  # finished rows are logged as -1
    tr = trace_from_accept_log(log, horizon=4)
    assert tr.count == int((log >= 0).sum()) and max(tr.samples) <= 4
    # injected law: l = min(trace sample, k) -> the censored mean matches the source trace's at s = 4
    assert abs(estimate_expected_correct(tr, 4) - estimate_expected_correct(example_trace(), 4)) < 0.6
