"""Shipped illustrative calibration / acceptance fixtures.

Same values as ``specbatch.presets`` (reference ``pkg/src/specbatch/presets.py:20-52``)
so that LUT / simulator known-answer tests carry over; the B200 engine
replaces the calibration with measured numbers (:mod:`.profiler`) and uses
:func:`example_trace` as the acceptance-injection law for random-weight
throughput runs.
"""

from __future__ import annotations

from .acceptance import AcceptanceTrace, PowerLawFit
from .cost_model import LinearStepModel

__all__ = ["example_calibration", "example_fit", "example_trace", "PRESET_NAME"]

PRESET_NAME = "rtx3090-like"

_SIZES = (1, 2, 4, 8, 16, 32)


def example_calibration() -> LinearStepModel:
    alpha = (0.35, 0.45, 0.60, 0.80, 1.00, 1.25)
    ssm = (0.08, 0.09, 0.10, 0.12, 0.15, 0.20)
    return LinearStepModel(alpha=dict(zip(_SIZES, alpha)), beta=5.0, ssm_step=dict(zip(_SIZES, ssm)))


def example_fit() -> PowerLawFit:
    return PowerLawFit(c=0.9, gamma=0.548)


def example_trace(n: int = 200, horizon: int = 80) -> AcceptanceTrace:
    """Deterministic trace whose censored means follow 0.9*s^0.548.

    Tail counts #{l_i >= k} = round(n*(l(k)-l(k-1))) for k=1..8; the count of
    samples >= 8 is spread evenly over [8, horizon-1].
    """
    f = example_fit()
    ge = [round(n * (f(1) if k == 1 else f(k) - f(k - 1))) for k in range(1, 9)]
    samples: list[int] = [0] * (n - ge[0])
    for v in range(1, 8):
        samples += [v] * (ge[v - 1] - ge[v])
    m = ge[7]
    samples += [8 + (j * (horizon - 9)) // max(m - 1, 1) for j in range(m)]
    return AcceptanceTrace(samples=tuple(samples), horizon=horizon)
