"""Error types of the drop-in API (same classes/bases as R/errors.py:4-13)."""


class ValidationError(ValueError):
    """An input violated a documented precondition (shape, spacing, bounds...)."""


class PrecisionError(ArithmeticError):
    """float64 cannot represent the result: some convolution value is <= 0.

    Messages name the remedy (more precision bits or a larger tau), exactly as
    the reference does, so callers matching on "precision" keep working.
    """


class NativeError(RuntimeError):
    """The CUDA library reported a device/runtime failure (C-ABI status 3)."""
