"""Error taxonomy of the drop-in API.

Mirrors the reference's exception classes (fftddm/errors.py:1-24) so that
callers catching `fftddm.errors.*` keep working.  The native library reports
failures as integer status codes (include/fftddm_b200.h, FD_ERR_*); the
loader in `_native.py` maps each code back onto one of these classes.
"""


class FftDdmError(Exception):
    """Root of every error raised by the package."""


class ValidationError(FftDdmError):
    """Structural problem with a subdomain, interface, field length or config."""


class SingularOperatorError(FftDdmError):
    """A per-mode tridiagonal pivot vanished (ref rectsolver.py:21,156-163)."""


class ConvergenceError(FftDdmError):
    """GMRES did not reach the tolerance; `.report` holds the SolveReport and
    `.solution` the last iterate (ref krylov.py:156-165)."""

    def __init__(self, message, report=None):
        super().__init__(message)
        self.report = report
        self.solution = None


class NativeError(FftDdmError):
    """CUDA / library failure inside the native extension."""
