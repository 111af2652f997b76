"""B200-native drop-in for the hot path of the FFT-preconditioned Schur/GMRES
Helmholtz-Poisson solver of arXiv 2509.23180 (reference package `fftddm`).

Public surface mirrors fftddm/__init__.py:15-31.  Host-side data model
(geometry) is pure Python; every solve/apply/transform runs in the sm_100a
library libfftddm_b200.so (csrc/), with torch CUDA tensors as buffers.
"""

from .errors import ConvergenceError, FftDdmError, SingularOperatorError, ValidationError
from .geometry import (BoundaryKind, CompositeDomain, GridField, Interface, RectSubdomain,
                       load_composite, make_interface, validate)

__version__ = "0.1.0"

_LAZY = {
    "plan_rect": "rectsolver", "solve_rect": "rectsolver", "lift_dirichlet": "rectsolver",
    "apply_rect_operator": "rectsolver", "solve_rect_batched": "rectsolver",
    "build_schur_operator": "ddm", "ddm_solve": "ddm",
    "GmresConfig": "krylov", "SolveReport": "krylov", "gmres": "krylov",
}


def __getattr__(name):
    if name in _LAZY:
        import importlib
        mod = importlib.import_module(f".{_LAZY[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)


__all__ = ["BoundaryKind", "CompositeDomain", "ConvergenceError", "FftDdmError", "GmresConfig",
           "GridField", "Interface", "RectSubdomain", "SolveReport", "SingularOperatorError",
           "ValidationError", "build_schur_operator", "ddm_solve", "gmres", "load_composite",
           "make_interface", "plan_rect", "solve_rect", "validate", "lift_dirichlet",
           "apply_rect_operator", "solve_rect_batched"]
