"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is importable there, not on the GPU
box):   python tests/golden/make_golden.py [/root/reference/pkg/src]

Outputs (committed, small):
  tokenlevel.json  -- run_batch(TokenLevel) traces recorded through the
                      reference's own TokenLevel/decode_step: per step and live
                      sequence the drafts it generated, the accepted length,
                      the advance, plus final token streams (pins K4/K5)
  engine.json      -- verify / decode_step / run_batch KATs and TraceSampler runs
  policy.json      -- analytic + simulated LUTs, lookup table, fixed policies
  serving.json     -- traffic generation + run_simulation reports
  cost_model.json  -- predict_runtime / delta / optimum values
  files/           -- the six file formats written by the reference's own
                      writers (trace CSV, LUT CSV, calibration JSON, workload
                      CSV, simulation records CSV, report JSON) plus a
                      step-sample CSV in the layout of its reader; pins the
                      byte format of our writers and our readers
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

import specbatch as sbr  # noqa: E402
from specbatch import engine as reng  # noqa: E402
from specbatch import policy as rpol  # noqa: E402
from specbatch import simulator as rsim  # noqa: E402
from specbatch import cost_model as rcm  # noqa: E402

OUT = Path(__file__).resolve().parent


def dump(name, obj):
    (OUT / name).write_text(json.dumps(obj, indent=1, sort_keys=True) + "\n")
    print("wrote", OUT / name)


class RecordingTokenLevel(reng.TokenLevel):
    """The reference TokenLevel, instrumented to log what it drafted."""

    def __init__(self, p_err, seed):
        super().__init__(p_err, seed)
        self.log = []

    def step(self, state, s, rng):
        if s == 0:
            acc = 0
            drafts = []
        else:
            drafts = self.draft_tokens(state, s, rng)
            target = [self.target_token(state.request_id, state.produced + i) for i in range(s)]
            acc = reng.verify(drafts, target)
        self.log.append({"rid": state.request_id, "produced": state.produced, "drafts": drafts,
                         "targets": [self.target_token(state.request_id, state.produced + i) for i in range(s + 1)],
                         "accepted": acc, "advanced": min(acc + 1, state.remaining)})
        return acc


def tokenlevel_cases():
    cases = []
    specs = [
        (4, 4, 37, 0.35, 7, 11), (8, 8, 64, 0.2, 3, 5), (3, 1, 20, 0.5, 1, 2), (5, 0, 9, 0.3, 2, 9),
        (16, 6, 48, 0.1, 9, 13), (2, 8, 128, 0.05, 4, 21), (7, 3, 33, 0.9, 5, 1), (1, 8, 1, 0.0, 0, 0),
    ]
    for b, s, n, p_err, seed, rng_seed in specs:
        oracle = RecordingTokenLevel(p_err, seed)
        states = [reng.SequenceState(request_id=100 * seed + i, target_len=n + (i % 3)) for i in range(b)]
        res = reng.run_batch(states, s, sbr.example_calibration(), oracle, np.random.default_rng(rng_seed))
        # regroup the flat log into steps: each step visits the then-live sequences in order
        steps, cur, seen = [], [], set()
        for rec in oracle.log:
            if rec["rid"] in seen:
                steps.append(cur)
                cur, seen = [], set()
            cur.append(rec)
            seen.add(rec["rid"])
        if cur:
            steps.append(cur)
        cases.append({
            "b": b, "s": s, "target_lens": [st.target_len for st in states], "p_err": p_err, "seed": seed,
            "rng_seed": rng_seed, "request_ids": [st.request_id for st in states], "steps": steps,
            "tokens": {str(st.request_id): st.tokens for st in states},
            "result": {"steps": res.steps, "total_time": res.total_time, "tokens_generated": res.tokens_generated,
                       "finish": {str(k): v for k, v in res.per_sequence_finish.items()}},
        })
    return cases


class ConstOracle(reng.DraftOracle):
    def __init__(self, a):
        self.a = a

    def step(self, state, s, rng):
        return min(self.a, s)


def engine_cases():
    out = {"verify": [], "decode_step": [], "run_batch_const": [], "trace_sampler": []}
    for d, t in [([5, 7, 3, 9], [5, 7, 9, 2]), ([1, 2, 3, 4], [1, 2, 3, 4]), ([1, 0, 0], [2, 0, 0]), ([], [])]:
        out["verify"].append({"draft": d, "target": t, "l": reng.verify(d, t)})
    for (tl, s, p_err) in [(8, 4, 0.0), (8, 4, 1.0), (3, 4, 0.0), (4, 0, 0.0)]:
        st = reng.SequenceState(request_id=0, target_len=tl)
        o = reng.decode_step(st, s, reng.TokenLevel(p_err=p_err), np.random.default_rng(1234))
        out["decode_step"].append({"target_len": tl, "s": s, "p_err": p_err, "accepted": o.accepted,
                                   "advanced": o.advanced, "tokens": st.tokens})
    simple = rcm.LinearStepModel(alpha={1: 1.0}, beta=5.0, ssm_step={1: 0.2})
    for n in (1, 5, 8, 17, 32):
        for s in range(0, 9):
            for a in sorted({0, s // 2, s}):
                r = reng.run_batch([reng.SequenceState(0, n)], s, simple, ConstOracle(a), np.random.default_rng(0))
                out["run_batch_const"].append({"n": n, "s": s, "a": a, "steps": r.steps, "total_time": r.total_time})
    cal, trace = sbr.example_calibration(), sbr.example_trace()
    for b, s, n, seed in [(4, 3, 32, 1234), (3, 4, 64, 99), (16, 4, 128, 7), (8, 0, 16, 5), (1, 8, 300, 0)]:
        states = [reng.SequenceState(request_id=i, target_len=n) for i in range(b)]
        r = reng.run_batch(states, s, cal, reng.TraceSampler(trace), np.random.default_rng(seed))
        out["trace_sampler"].append({"b": b, "s": s, "n": n, "seed": seed, "steps": r.steps,
                                     "total_time": r.total_time,
                                     "finish": {str(k): v for k, v in r.per_sequence_finish.items()}})
    return out


def policy_cases():
    cal, trace, fit = sbr.example_calibration(), sbr.example_trace(), sbr.example_fit()
    ref_lut = rpol.SpeculationLUT(entries={1: 6, 2: 5, 4: 4, 8: 3, 16: 2, 32: 2}, s_grid=tuple(range(9)))
    out = {
        "analytic_trace": rpol.build_lut(cal, trace).entries,
        "analytic_fit": rpol.build_lut(cal, fit).entries,
        "simulated_seed1": rpol.build_lut(cal, trace, mode="simulated", sample_size=200,
                                          rng=np.random.default_rng(1)).entries,
        "simulated_seed7_small": rpol.build_lut(cal, trace, mode="simulated", sample_size=40,
                                                profiled_sizes=(1, 4, 16), rng=np.random.default_rng(7)).entries,
        "lookup": [[b, rpol.lookup(ref_lut, b).chosen_s, rpol.lookup(ref_lut, b).source] for b in range(1, 100)],
    }
    rng = np.random.default_rng(1234)
    rand = []
    sizes = (1, 2, 4, 8, 16, 32)
    for _ in range(50):
        slopes = np.cumsum(rng.uniform(0.05, 0.8, size=len(sizes)))
        ssm = np.cumsum(rng.uniform(0.01, 0.1, size=len(sizes)))
        beta = float(rng.uniform(0.0, 10.0))
        c, g = float(rng.uniform(0.3, 2.0)), float(rng.uniform(0.1, 0.9))
        model = rcm.LinearStepModel(alpha=dict(zip(sizes, map(float, slopes))), beta=beta,
                                    ssm_step=dict(zip(sizes, map(float, ssm))))
        lut = rpol.build_lut(model, sbr.PowerLawFit(c=c, gamma=g), profiled_sizes=sizes)
        rand.append({"alpha": list(map(float, slopes)), "ssm": list(map(float, ssm)), "beta": beta, "c": c,
                     "gamma": g, "lut": lut.entries})
    out["random_calibrations"] = rand
    return json.loads(json.dumps(out))


def serving_cases():
    cal, trace = sbr.example_calibration(), sbr.example_trace()
    lut = rpol.build_lut(cal, trace)
    out = []
    for name, wl_fn, pol in [
        ("poisson_fixed2", lambda r: sbr.gen_arrivals(sbr.TrafficConfig(0.05, 1.0, 120), r), sbr.fixed_policy(2)),
        ("poisson_adaptive", lambda r: sbr.gen_arrivals(sbr.TrafficConfig(0.05, 1.0, 120), r),
         sbr.AdaptivePolicy(lut)),
        ("bursty_none", lambda r: sbr.gen_arrivals(sbr.TrafficConfig(0.02, 5.0, 200), r), sbr.fixed_policy(0)),
        ("phased_adaptive", lambda r: sbr.gen_phased(sbr.PhaseSchedule(phases=(
            (5.0, sbr.TrafficConfig(0.02, 1.0, 10**6)), (5.0, sbr.TrafficConfig(0.2, 1.0, 10**6)))), r),
         sbr.AdaptivePolicy(lut)),
    ]:
        wl = wl_fn(np.random.default_rng(42))
        rep = rsim.run_simulation(wl, rsim.ServerConfig(policy=pol, max_batch=16), cal, trace,
                                  np.random.default_rng(3))
        out.append({"name": name, "arrivals": [r.arrival for r in wl], "ids": [r.id for r in wl],
                    "avg_latency": rep.avg_latency, "timeline": [list(t) for t in rep.timeline],
                    "records": [[r.request_id, r.t_a, r.t_start, r.t_b, r.latency, r.served_batch_size, r.used_s]
                                for r in rep.records], "policy": rep.policy})
    return out


def cost_cases():
    cal, fit = sbr.example_calibration(), sbr.example_fit()
    out = {"predict": [], "delta": [], "root": None, "discrete": []}
    for b in (1, 3, 8, 32, 50):
        for s in range(0, 9):
            p = rcm.predict_runtime(cal, fit, 128, b, s)
            out["predict"].append([b, s, p.T_L, p.T_S, p.T_total, p.expected_steps, p.per_token])
    prm = rcm.OptimalityParams(alpha_eff=1.0, beta=5.0, c=0.9, gamma=0.548)
    out["delta"] = [[s, rcm.eval_delta(prm, s)] for s in (0.5, 1, 2, 3, 4.5, 8)]
    out["root"] = rcm.optimal_speculation_continuous(prm, 1, 8, tol=1e-7)
    out["discrete"] = [[b, rcm.optimal_speculation_discrete(cal, fit, 128, b, range(9))] for b in (1, 2, 4, 8, 16, 32)]
    # OLS fits of step samples (cost_model.py:145-170) and the acceptance power law (acceptance.py:85-106)
    rng = np.random.default_rng(11)
    fits = []
    for b in (1, 4, 16):
        ys = [float(2.5 + 0.03 * b * s + rng.normal(0, 0.01)) for s in range(1, 9)]
        smp = [rcm.StepTimeSample(batch_size=b, query_len=s, measured_time=y) for s, y in zip(range(1, 9), ys)]
        fits.append([b, ys, list(rcm.fit_linear_step_time(smp))])
    out["fit_linear"] = fits
    from specbatch import acceptance as racc
    trace = sbr.example_trace()
    pts = [(s, racc.estimate_expected_correct(trace, s)) for s in range(1, 9)]
    pl = racc.fit_power_law(pts)
    out["power_law"] = {"points": [list(p) for p in pts], "c": pl.c, "gamma": pl.gamma}
    return out


def file_cases():
    from specbatch import acceptance as racc, traffic as rtr

    d = OUT / "files"
    d.mkdir(exist_ok=True)
    cal, fit, trace = sbr.example_calibration(), sbr.example_fit(), sbr.example_trace()
    racc.save_trace(trace, d / "trace.csv")
    lut = rpol.build_lut(cal, trace)
    rpol.save_lut(lut, d / "lut.csv", seed=7, calibration="example")
    rcm.save_calibration(cal, d / "calibration.json", fit=fit)
    rcm.save_calibration(cal, d / "calibration_nofit.json")
    wl = sbr.gen_arrivals(sbr.TrafficConfig(0.05, 1.0, 30), np.random.default_rng(42))
    rtr.save_workload(wl, d / "workload.csv")
    rep = rsim.run_simulation(wl, rsim.ServerConfig(policy=sbr.AdaptivePolicy(lut), max_batch=16, seed=3), cal,
                              trace, np.random.default_rng(3))
    rsim.save_records(rep, d / "records.csv")
    rsim.save_report(rep, d / "report.json")
    # the reference reads step samples (cost_model.py:302-314) but has no writer: csv.writer layout
    import csv
    with open(d / "step_samples.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["batch_size", "query_len", "time_ms"])
        for b, sl, ms in [(1, 1, 3.25), (1, 8, 3.875), (8, 3, 3.5), (64, 1, 7.015625)]:
            w.writerow([b, sl, repr(ms)])
    samples = rcm.load_step_samples(d / "step_samples.csv")
    (d / "expected.json").write_text(json.dumps({
        "lut_entries": {str(b): v for b, v in lut.entries.items()},
        "samples": [[x.batch_size, x.query_len, x.measured_time] for x in samples],
        "workload": [[r.id, r.arrival, r.gen_len] for r in rtr.load_workload(d / "workload.csv")],
        "avg_latency": rep.avg_latency, "policy": rep.policy,
    }, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    file_cases()
    dump("tokenlevel.json", tokenlevel_cases())
    dump("engine.json", engine_cases())
    dump("policy.json", policy_cases())
    dump("serving.json", serving_cases())
    dump("cost_model.json", cost_cases())
