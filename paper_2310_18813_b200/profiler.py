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

__all__ = ["measure_step_samples", "calibrate", "model_from_samples"]

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
