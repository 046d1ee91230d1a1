"""Exception types mirroring hx/errors.py:4-25 for the hot path."""


class FactorizationError(RuntimeError):
    """A dense restricted block was not SPD (hx/sparse.py:87-98)."""


class ConvergenceError(RuntimeError):
    """Raised when an iterative solve fails inside a transient sequence."""

    def __init__(self, message, report=None):
        super().__init__(message)
        self.report = report
