"""Exception types of the reference (core.py:24-29), re-declared so callers can
catch the same classes on the GPU path."""


class ShapeError(ValueError):
    """An array shape is inconsistent with the scan's contract (core.py:24-25)."""


class NonFiniteError(ValueError):
    """An externally supplied array contains NaN or Inf (core.py:28-29)."""
