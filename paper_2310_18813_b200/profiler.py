"""Measured calibration of the cost model on this B200 (the paper's offline
profiling step; reference formats cost_model.py:273-314).

``calibrate(engine)`` times the real verify forward at every (b, s) cell and
one draft decode step per b with CUDA events (graph-replayed, warm), emits
the reference's ``StepTimeSample`` rows (query_len = s, the reference's
convention for a verify of s drafted tokens -- the kernels process s+1), and
fits them with the reference's own OLS (``fit_linear_step_time``) into a
``LinearStepModel`` that ``build_lut`` / ``run_simulation`` consume unchanged.
"""

from __future__ import annotations

import warnings

import numpy as np

from .cost_model import LinearStepModel, StepTimeSample, fit_linear_step_time
from .errors import CalibrationWarning

__all__ = ["measure_step_samples", "calibrate", "model_from_samples", "table_lut", "measure_cost_table", "dense_tables"]

_MIN_SLOPE = 1e-4  # ms per token; LinearStepModel requires alpha > 0


def measure_step_samples(engine, batch_sizes=(1, 2, 4, 8), k_grid=range(1, 9), ctx: int | None = None, reps: int = 10):
    ctx = ctx or (engine.prompt_len + engine.max_new // 2)
    samples, ssm = [], {}
    for b in batch_sizes:
        for s in k_grid:
            ms = engine.time_verify(b, s, ctx=ctx, reps=reps)
            samples.append(StepTimeSample(batch_size=b, query_len=s, measured_time=ms))
        ssm[b] = engine.time_draft_step(b, ctx=ctx, reps=reps)
    return samples, ssm


def model_from_samples(samples, ssm: dict) -> LinearStepModel:
    """Per-b OLS slopes; the shared intercept is the mean of per-b intercepts.
    Tables are made non-decreasing in b (cumulative max) and strictly positive,
    as LinearStepModel requires (cost_model.py:59-85)."""
    by_b: dict[int, list] = {}
    for smp in samples:
        by_b.setdefault(smp.batch_size, []).append(smp)
    alpha, inter = {}, []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", CalibrationWarning)
        for b in sorted(by_b):
            slope, icpt = fit_linear_step_time(by_b[b])
            alpha[b] = slope
            inter.append(icpt)
    run = _MIN_SLOPE
    for b in sorted(alpha):
        run = max(run, alpha[b])
        alpha[b] = run
    run = 1e-6
    ssm_t = {}
    for b in sorted(ssm):
        run = max(run, float(ssm[b]))
        ssm_t[b] = run
    beta = max(0.0, float(np.mean(inter)))
    return LinearStepModel(alpha=alpha, beta=beta, ssm_step=ssm_t)


def calibrate(engine, batch_sizes=(1, 2, 4, 8), k_grid=range(1, 9), ctx: int | None = None, reps: int = 10):
    samples, ssm = measure_step_samples(engine, batch_sizes, k_grid, ctx, reps)
    return model_from_samples(samples, ssm), samples


def table_lut(verify_ms: dict, draft_ms: dict, trace, s_grid=range(9), profiled_sizes=(1, 2, 4, 8, 16),
              sample_size: int = 200, rng=None, gen_len: int = 128):
    """b -> k LUT from the MEASURED cost table instead of the linear fit.

    ``verify_ms[(b, s)]`` is the measured verify forward at speculation length s
    (s + 1 query tokens per sequence, s = 0 included) and ``draft_ms[b]`` one
    draft step.  Step counts come from the reference's own simulated procedure
    (run_batch over TraceSampler, policy.py:110-123: a formed batch runs until
    its LAST sequence finishes); each step is charged verify_ms[(b, s)] +
    s * draft_ms[b].  This isolates the two things the analytic LUT
    (policy.py:101-105) does not see on B200: t_L(b, s) is step-shaped in the
    token count b(s+1) (GEMM token tiles), not linear, and the batch is held
    for its slowest sequence (max over b of the step counts, not N / (E[l]+1)).
    Returns (SpeculationLUT, {(b, s): ms per token})."""
    from .policy import SpeculationLUT

    entries, cells = _formed_table(verify_ms, draft_ms, trace, s_grid, profiled_sizes, sample_size, rng, gen_len)
    grid = tuple(sorted(set(s_grid)))
    return SpeculationLUT(entries=entries, s_grid=grid, provenance={"mode": "table-simulated"}), cells


def _formed_table(verify_ms, draft_ms, trace, s_grid, sizes, sample_size, rng, gen_len):
    """argmin_s of ms per token for a batch held until its last sequence finishes:
    step counts from the reference's run_batch over TraceSampler (policy.py:110-123),
    each step charged verify_ms[(b, s)] + s * draft_ms[b].  Ties -> smaller s."""
    from .engine import SequenceState, TraceSampler, run_batch

    rng = rng if rng is not None else np.random.default_rng(0)
    unit = LinearStepModel(alpha={1: 1e-300}, beta=1.0, ssm_step={1: 1e-300})  # per-step cost ~1: counts steps
    grid = tuple(sorted(set(s_grid)))
    entries, cells = {}, {}
    for b in sorted(sizes):
        best, best_t = None, float("inf")
        for s in grid:
            steps = toks = 0
            for j in range(-(-sample_size // b)):
                states = [SequenceState(request_id=j * b + i, target_len=gen_len) for i in range(b)]
                res = run_batch(states, s, unit, TraceSampler(trace), rng)
                steps += res.steps
                toks += res.tokens_generated
            t = steps * (verify_ms[(b, s)] + s * draft_ms[b]) / toks
            cells[(b, s)] = t
            if t < best_t:
                best, best_t = s, t
        entries[b] = best
    return entries, cells


def measure_cost_table(engine, batch_sizes, k_grid=range(9), ctx: int | None = None, reps: int = 10):
    """Measured verify forward ms at every (b, s) (s + 1 query tokens per sequence,
    s = 0 included) and one draft step's ms per b, graph-replayed with CUDA events."""
    ctx = ctx or (engine.prompt_len + engine.max_new // 2)
    verify_ms = {(b, s): engine.time_verify(b, s, ctx=ctx, reps=reps) for b in batch_sizes for s in k_grid}
    draft_ms = {b: engine.time_draft_step(b, ctx=ctx, reps=reps) for b in batch_sizes}
    return verify_ms, draft_ms


def dense_tables(verify_ms: dict, draft_ms: dict, trace, sizes, s_grid=range(9), sample_size: int = 200, rng=None,
                 gen_len: int = 128):
    """b -> s tables at EVERY size in `sizes` (for policy.DensePolicy) from a measured cost table.

    ``formed``: a formed batch held until its slowest sequence finishes (the
    reference's execution model, engine.py:186-188) -- as :func:`table_lut`.
    ``continuous``: continuous batching retires each sequence as it finishes, so
    an iteration is worth b * (E[min(l, s)] + 1) tokens (E = the trace's
    censored mean, acceptance.py Eq. 4) and costs verify_ms[(b, s)] + s *
    draft_ms[b]; the table keeps argmin_s of ms per token (ties -> smaller s).
    Returns (formed, continuous, {"formed": cells, "continuous": cells})."""
    from .acceptance import estimate_expected_correct

    formed, fcells = _formed_table(verify_ms, draft_ms, trace, s_grid, sizes, sample_size, rng, gen_len)
    grid = tuple(sorted(set(s_grid)))
    el = {s: (estimate_expected_correct(trace, min(s, trace.horizon)) if s else 0.0) for s in grid}
    cont, ccells = {}, {}
    for b in sorted(sizes):
        best, best_t = None, float("inf")
        for s in grid:
            t = (verify_ms[(b, s)] + s * draft_ms[b]) / (b * (el[s] + 1.0))
            ccells[(b, s)] = t
            if t < best_t:
                best, best_t = s, t
        cont[b] = best
    return formed, cont, {"formed": fcells, "continuous": ccells}
