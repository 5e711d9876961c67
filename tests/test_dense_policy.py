"""DensePolicy and the dense b -> s tables (profiler.dense_tables): the
extension that profiles every live batch size instead of the reference's
powers of two (policy.py:131-150 resolves 9..15 to min(s_8, s_16))."""

import numpy as np
import pytest

from paper_2310_18813_b200.acceptance import estimate_expected_correct
from paper_2310_18813_b200.policy import AdaptivePolicy, DensePolicy, SpeculationLUT
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.profiler import dense_tables, table_lut
from paper_2310_18813_b200.simulator import ServerConfig, run_simulation
from paper_2310_18813_b200.cost_model import LinearStepModel
from paper_2310_18813_b200.traffic import Request


def _costs(sizes):
    # flat verify up to 64 tokens, then linear in the token count; draft step grows slowly with b
    vm = {(b, s): 2.7 + 0.002 * b * (s + 1) + 0.02 * max(0, b * (s + 1) - 64) for b in sizes for s in range(9)}
    dm = {b: 0.05 + 0.001 * b for b in sizes}
    return vm, dm


def test_dense_policy_lookup():
    pol = DensePolicy({1: 8, 2: 7, 4: 5, 16: 3})
    assert pol.label == "adaptive-dense"
    assert pol.decide(1).chosen_s == 8 and pol.decide(1).source == "lut-exact"
    assert pol.decide(3).chosen_s == 7 and pol.decide(3).source == "lut-clamped"  # largest profiled size below
    assert pol.decide(15).chosen_s == 5
    assert pol.decide(40).chosen_s == 3
    with pytest.raises(ValueError):
        pol.decide(0)
    with pytest.raises(ValueError):
        DensePolicy({})
    # the reference rule on the same powers of two picks the smaller neighbour in between
    ref = AdaptivePolicy(SpeculationLUT(entries={1: 8, 2: 7, 4: 5, 16: 3}, s_grid=tuple(range(9))))
    assert ref.decide(3).chosen_s == 5 and ref.decide(15).chosen_s == 3


def test_dense_tables_match_table_lut_and_closed_form():
    tr = example_trace()
    sizes = range(1, 17)
    vm, dm = _costs(sizes)
    formed, cont, cells = dense_tables(vm, dm, tr, sizes, sample_size=64, rng=np.random.default_rng(5))
    assert sorted(formed) == list(sizes) and sorted(cont) == list(sizes)
    # formed table on the powers of two == table_lut with the same rng stream
    lut, _ = table_lut(vm, dm, tr, profiled_sizes=(1, 2, 4, 8, 16), sample_size=64, rng=np.random.default_rng(5))
    f2, _, _ = dense_tables(vm, dm, tr, (1, 2, 4, 8, 16), sample_size=64, rng=np.random.default_rng(5))
    assert f2 == lut.entries
    # continuous table: argmin of (verify + s * draft) / (b (E[min(l, s)] + 1)), ties -> smaller s
    for b in sizes:
        t = [(vm[(b, s)] + s * dm[b]) / (b * ((estimate_expected_correct(tr, s) if s else 0.0) + 1)) for s in range(9)]
        assert cont[b] == int(np.argmin(t))
        assert cells["continuous"][(b, cont[b])] == pytest.approx(min(t))
    # larger batches never want longer speculation under this cost shape
    assert cont[16] <= cont[8] <= cont[1]


def test_dense_policy_drives_the_simulator():
    model = LinearStepModel(alpha={1: 0.01, 16: 0.02}, beta=2.7, ssm_step={1: 0.05, 16: 0.06})
    wl = [Request(id=i, arrival=0.01 * i, gen_len=32) for i in range(40)]
    rep = run_simulation(wl, ServerConfig(policy=DensePolicy({b: 4 for b in range(1, 17)}), max_batch=16), model,
                         example_trace(), np.random.default_rng(0))
    assert rep.policy == "adaptive-dense"
    assert all(r.used_s == 4 for r in rep.records)


def test_measure_cost_table_calls_engine_per_cell():
    from paper_2310_18813_b200.profiler import measure_cost_table

    class FakeEngine:
        prompt_len, max_new = 128, 128

        def __init__(self):
            self.calls = []

        def time_verify(self, b, k, ctx, reps):
            self.calls.append(("v", b, k, ctx))
            return 2.7 + 0.01 * b * (k + 1)

        def time_draft_step(self, b, ctx, reps):
            self.calls.append(("d", b, ctx))
            return 0.05 + 0.001 * b

    eng = FakeEngine()
    vm, dm = measure_cost_table(eng, range(1, 4), k_grid=range(3))
    assert sorted(vm) == [(b, k) for b in range(1, 4) for k in range(3)]
    assert sorted(dm) == [1, 2, 3]
    assert vm[(2, 1)] == pytest.approx(2.74) and dm[3] == pytest.approx(0.053)
    assert all(c[-1] == 192 for c in eng.calls)  # default context: prompt + half the generation
