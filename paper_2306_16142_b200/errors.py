"""Exception classes mirroring ddfield/errors.py:8-17.

When the reference package is importable the classes subclass its own, so
code written against ``ddfield.errors`` catches errors raised here unchanged.
"""

try:  # pragma: no cover - depends on the environment
    from ddfield import errors as _ref
    _BASE, _DATA, _NUM = _ref.DdfError, _ref.DataError, _ref.NumericError
except Exception:  # the GPU box has no reference
    _BASE = _DATA = _NUM = Exception


class DdfError(_BASE):
    """Base class for all toolkit errors."""


class DataError(DdfError, _DATA):
    """Unreadable, malformed, or inconsistent input data."""


class NumericError(DdfError, _NUM):
    """Numerical failure (normal sign rule, degenerate gradient)."""
