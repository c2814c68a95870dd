"""Typed errors with the reference's names (errors.py:8-50 of the reference).

When the reference package `ivhd` is importable in the same interpreter, each
class also derives from its reference namesake, so callers that catch
`ivhd.errors.IvhdError` (e.g. the reference CLI, cli.py:28-37) keep working
when `run_embedding` points at this package.
"""

try:  # optional: only for drop-in exception compatibility
    from ivhd import errors as _ref  # type: ignore
except Exception:  # pragma: no cover - reference not installed
    _ref = None


def _bases(name, *own):
    extra = getattr(_ref, name, None) if _ref is not None else None
    if extra is None:
        return own
    if own == (Exception,):
        return (extra,)
    return own + (extra,)


class IvhdError(*_bases("IvhdError", Exception)):
    """Base class for every error raised by this package."""


class InvalidArgumentError(*_bases("InvalidArgumentError", IvhdError)):
    """An argument is outside its documented domain."""


class DimensionMismatchError(*_bases("DimensionMismatchError", IvhdError)):
    """Shapes or widths are inconsistent."""


class DeviceError(IvhdError):
    """The CUDA library failed (or is missing on this machine)."""


class NumericalDivergenceError(*_bases("NumericalDivergenceError", IvhdError)):
    """Non-finite coordinates; carries the last finite state
    (reference errors.py:40-50, engine.py:373-377)."""

    def __init__(self, iteration, state=None):
        Exception.__init__(self, f"embedding diverged at iteration {iteration}")
        self.iteration = iteration
        self.state = state


class DegenerateMetricError(*_bases("DegenerateMetricError", IvhdError)):
    """The metric cannot be evaluated on a row (zero-norm vector under cosine;
    reference errors.py:30-38)."""

    def __init__(self, message, row=None):
        if row is not None:
            message = f"{message} (row {row})"
        Exception.__init__(self, message)
        self.row = row


class MalformedInputError(*_bases("MalformedInputError", IvhdError)):
    """A file failed to parse (reference errors.py:12-20)."""

    def __init__(self, message, row=None):
        if row is not None:
            message = f"{message} (row {row})"
        Exception.__init__(self, message)
        self.row = row
