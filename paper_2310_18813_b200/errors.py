"""Error taxonomy of the drop-in API.

Mirrors the exception classes the reference raises so that callers catching
``specbatch`` errors keep working (reference: ``pkg/src/specbatch/errors.py:4-32``).
Native (C-ABI) failures surface as :class:`NativeError`, a ``RuntimeError``.
"""


class SpecbatchError(Exception):
    """Root of every model/configuration error (errors.py:4-5)."""


class DegenerateFitError(SpecbatchError):
    """A regression saw too few distinct abscissae (errors.py:8-9)."""


class UnfittableError(SpecbatchError):
    """No usable points survive the filters of a fit (errors.py:12-13)."""


class UncalibratedBatchError(SpecbatchError):
    """Batch size outside the calibrated table with interpolation off (errors.py:16-19)."""


class HorizonError(SpecbatchError):
    """Speculation length past the acceptance trace horizon (errors.py:22-25)."""


class ConfigError(SpecbatchError):
    """Invalid experiment / server / engine configuration (errors.py:28-29)."""


class CalibrationWarning(UserWarning):
    """Suspicious but non-fatal calibration result (errors.py:30-32)."""


class NativeError(RuntimeError):
    """A C-ABI entry point returned a non-zero CUDA / library status."""

    def __init__(self, fn: str, code: int, msg: str = ""):
        self.fn = fn
        self.code = code
        super().__init__(f"{fn} failed with status {code}{': ' + msg if msg else ''}")
