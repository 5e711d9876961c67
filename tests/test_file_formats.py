"""The reference's file formats (calibration JSON cost_model.py:273-299,
step-sample CSV cost_model.py:302-314, trace CSV acceptance.py:120-145, LUT CSV
policy.py:188-213, workload CSV traffic.py:126-145, simulation records / report
simulator.py:156-186).  Fixtures under tests/golden/files/ were written by the
reference's OWN writers (tests/golden/make_golden.py::file_cases); our writers
must reproduce them byte for byte and our readers must parse them.  When the
reference install (baseline/_ref) is present, its readers also parse ours."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2310_18813_b200 import (AdaptivePolicy, ServerConfig, build_lut, example_calibration, example_fit,
                                   example_trace, run_simulation)
from paper_2310_18813_b200.acceptance import load_trace, save_trace, trace_from_accept_log
from paper_2310_18813_b200.cost_model import (StepTimeSample, load_calibration, load_step_samples,
                                              save_calibration, save_step_samples)
from paper_2310_18813_b200.policy import load_lut, save_lut
from paper_2310_18813_b200.simulator import save_records, save_report
from paper_2310_18813_b200.traffic import TrafficConfig, gen_arrivals, load_workload, save_workload

FILES = Path(__file__).resolve().parent / "golden" / "files"
REF_INSTALL = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def expected():
    return json.loads((FILES / "expected.json").read_text())


def _same_bytes(tmp_path, name, write):
    out = tmp_path / name
    write(out)
    assert out.read_bytes() == (FILES / name).read_bytes(), name


def test_trace_csv_bytes_and_roundtrip(tmp_path):
    _same_bytes(tmp_path, "trace.csv", lambda p: save_trace(example_trace(), p))
    assert b"\r\n" in (FILES / "trace.csv").read_bytes()  # csv.writer rows, as the reference writes them
    assert load_trace(FILES / "trace.csv") == example_trace()


def test_lut_csv_bytes_and_roundtrip(tmp_path, expected):
    lut = build_lut(example_calibration(), example_trace())
    assert {str(b): v for b, v in lut.entries.items()} == expected["lut_entries"]
    _same_bytes(tmp_path, "lut.csv", lambda p: save_lut(lut, p, seed=7, calibration="example"))
    back = load_lut(FILES / "lut.csv")
    assert back.entries == lut.entries
    assert back.provenance["seed"] == "7" and back.provenance["calibration"] == "example"


def test_calibration_json_bytes_and_roundtrip(tmp_path):
    cal, fit = example_calibration(), example_fit()
    _same_bytes(tmp_path, "calibration.json", lambda p: save_calibration(cal, p, fit=fit))
    _same_bytes(tmp_path, "calibration_nofit.json", lambda p: save_calibration(cal, p))
    m, f = load_calibration(FILES / "calibration.json")
    assert m == cal and f == fit
    m2, f2 = load_calibration(FILES / "calibration_nofit.json")
    assert m2 == cal and f2 is None


def test_step_samples_csv(tmp_path, expected):
    got = load_step_samples(FILES / "step_samples.csv")
    assert [[s.batch_size, s.query_len, s.measured_time] for s in got] == expected["samples"]
    _same_bytes(tmp_path, "step_samples.csv", lambda p: save_step_samples(got, p))


def test_workload_csv_bytes_and_roundtrip(tmp_path, expected):
    wl = gen_arrivals(TrafficConfig(0.05, 1.0, 30), np.random.default_rng(42))
    _same_bytes(tmp_path, "workload.csv", lambda p: save_workload(wl, p))
    back = load_workload(FILES / "workload.csv")
    assert [[r.id, r.arrival, r.gen_len] for r in back] == expected["workload"]


def test_simulation_records_and_report_bytes(tmp_path, expected):
    cal, trace = example_calibration(), example_trace()
    lut = build_lut(cal, trace)
    wl = gen_arrivals(TrafficConfig(0.05, 1.0, 30), np.random.default_rng(42))
    rep = run_simulation(wl, ServerConfig(policy=AdaptivePolicy(lut), max_batch=16, seed=3), cal, trace,
                         np.random.default_rng(3))
    assert rep.avg_latency == expected["avg_latency"] and rep.policy == expected["policy"]
    _same_bytes(tmp_path, "records.csv", lambda p: save_records(rep, p))
    _same_bytes(tmp_path, "report.json", lambda p: save_report(rep, p))


def test_trace_from_accept_log_drops_finished_rows():
    """the engine's accept log marks finished rows -1."""
    log = np.array([[3, 1, 0], [2, -1, 3], [-1, -1, 1]], dtype=np.int32)
    tr = trace_from_accept_log(log, horizon=3)
    assert tr.samples == (3, 1, 0, 2, 3, 1) and tr.horizon == 3
    with pytest.raises(ValueError):
        trace_from_accept_log(np.full((2, 2), -1), horizon=3)


@pytest.mark.skipif(not (REF_INSTALL / "specbatch").exists(), reason="reference install (baseline/_ref) absent")
def test_reference_readers_parse_our_files(tmp_path):
    sys.path.insert(0, str(REF_INSTALL))
    try:
        from specbatch import acceptance as racc, cost_model as rcm, policy as rpol, traffic as rtr
    finally:
        sys.path.remove(str(REF_INSTALL))
    cal, fit, trace = example_calibration(), example_fit(), example_trace()
    save_trace(trace, tmp_path / "t.csv")
    assert racc.load_trace(tmp_path / "t.csv").samples == trace.samples
    lut = build_lut(cal, trace)
    save_lut(lut, tmp_path / "l.csv", seed=1, calibration="x")
    assert rpol.load_lut(tmp_path / "l.csv").entries == lut.entries
    save_calibration(cal, tmp_path / "c.json", fit=fit)
    m, f = rcm.load_calibration(tmp_path / "c.json")
    assert dict(m.alpha) == dict(cal.alpha) and m.beta == cal.beta and (f.c, f.gamma) == (fit.c, fit.gamma)
    smp = [StepTimeSample(1, 2, 3.5), StepTimeSample(8, 3, 4.25)]
    save_step_samples(smp, tmp_path / "s.csv")
    assert [(x.batch_size, x.query_len, x.measured_time) for x in rcm.load_step_samples(tmp_path / "s.csv")] == \
        [(1, 2, 3.5), (8, 3, 4.25)]
    wl = gen_arrivals(TrafficConfig(0.05, 1.0, 10), np.random.default_rng(1))
    save_workload(wl, tmp_path / "w.csv")
    assert [(r.id, r.arrival, r.gen_len) for r in rtr.load_workload(tmp_path / "w.csv")] == \
        [(r.id, round(r.arrival, 9), r.gen_len) for r in wl]
