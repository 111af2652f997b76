"""ctypes binding of libfftddm_b200.so (include/fftddm_b200.h).

The extension is mandatory: importing a GPU entry point without the built
library, or without CUDA, raises NativeError.  There is no CPU fallback.
Status codes map onto the reference's exception classes (fftddm/errors.py).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (ConvergenceError, NativeError, SingularOperatorError,
                     ValidationError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfftddm_b200.so")

FD_OK, FD_ERR_VALIDATION, FD_ERR_SINGULAR, FD_ERR_NOT_CONVERGED, FD_ERR_CUDA, FD_ERR_UNSUPPORTED = range(6)

# every symbol the header declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "fd_last_error", "fd_version", "fd_plan_create", "fd_plan_create_axis", "fd_plan_create_ex", "fd_plan_create_sweep",
    "fd_plan_singular_modes", "fd_plan_set_pinv",
    "fd_transform_kind", "fd_transform_kind_pair",
    "fd_plan_destroy", "fd_plan_info",
    "fd_factor_tables_host", "fd_rect_solve", "fd_rect_solve_batched", "fd_dst_rows",
    "fd_transform_rows", "fd_assemble_rhs", "fd_stencil_apply", "fd_stencil_apply_ex", "fd_schur_create", "fd_schur_destroy", "fd_schur_apply",
    "fd_center_solve", "fd_precond_apply", "fd_unprecond_apply", "fd_gmres_precond",
    "fd_ddm_solve", "fd_schur_set_steklov", "fd_schur_use_steklov", "fd_arnoldi_step", "fd_basis_update", "fd_axpby", "fd_norm", "fd_dot",
    "fd_comm_unique_id", "fd_comm_init", "fd_comm_init_loopback", "fd_comm_rank", "fd_comm_destroy",
    "fd_schur_set_comm", "fd_ddm_solve_dist", "fd_schur_set_stencil",
)


class UnsupportedError(ValidationError, NotImplementedError):
    """Configuration outside the GPU path (NN/PP transform axis, transposed axis,
    transform lengths without a kernel)."""


class FdReport(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int), ("iterations", ctypes.c_int),
                ("restarts", ctypes.c_int), ("hist_len", ctypes.c_int),
                ("wall_time", ctypes.c_double), ("true_residual", ctypes.c_double)]


_lib = None
_lock = threading.Lock()
P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double
DP = ctypes.POINTER(ctypes.c_double)


def _declare(lib):
    sig = {
        "fd_last_error": (ctypes.c_char_p, []),
        "fd_version": (I, []),
        "fd_plan_create": (I, [ctypes.POINTER(P), I, I, D, D, D, D, D, I]),
        "fd_plan_create_axis": (I, [ctypes.POINTER(P), I, I, D, D, D, D, D, D, D, I, I]),
        "fd_transform_kind": (I, [I]),
        "fd_plan_create_ex": (I, [ctypes.POINTER(P), I, I, D, D, D, D, D, D, D, I, I, I]),
        "fd_plan_create_sweep": (I, [ctypes.POINTER(P), I, I, D, D, D, D, D, D, D, I, I, I, I, I]),
        "fd_plan_singular_modes": (I, [P, ctypes.POINTER(I), I, ctypes.POINTER(I)]),
        "fd_plan_set_pinv": (I, [P, I, ctypes.POINTER(D)]),
        "fd_transform_kind_pair": (I, [I, I]),
        "fd_plan_destroy": (I, [P]),
        "fd_plan_info": (I, [P, ctypes.POINTER(I), ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(I)]),
        "fd_factor_tables_host": (I, [I, I, D, D, D, D, D, DP, DP]),
        "fd_rect_solve": (I, [P, P, P, P]),
        "fd_rect_solve_batched": (I, [I, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P), P]),
        "fd_dst_rows": (I, [I, I, P, P, I, P]),
        "fd_transform_rows": (I, [I, I, I, I, P, P, I, P]),
        "fd_assemble_rhs": (I, [I, I, D, D, D, D, D, I, D, D, D, D, P, P, P]),
        "fd_stencil_apply": (I, [I, I, D, D, D, D, D, D, D, P, P, P]),
        "fd_stencil_apply_ex": (I, [I, I, D, D, D, D, D, D, D, I, I, P, P, P]),
        "fd_schur_create": (I, [ctypes.POINTER(P), P, D, D, I, ctypes.POINTER(P), ctypes.POINTER(I),
                                ctypes.POINTER(P), ctypes.POINTER(P), DP,
                                ctypes.POINTER(P), ctypes.POINTER(P), DP]),
        "fd_schur_destroy": (I, [P]),
        "fd_schur_set_steklov": (I, [P, I, I, I, D, D, D, D, D, I, P, P]),
        "fd_schur_use_steklov": (I, [P, I]),
        "fd_schur_apply": (I, [P, P, P, P]),
        "fd_center_solve": (I, [P, P, P, P]),
        "fd_precond_apply": (I, [P, P, P, P]),
        "fd_unprecond_apply": (I, [P, P, P, P]),
        "fd_gmres_precond": (I, [P, P, P, I, I, D, I, DP, I, ctypes.POINTER(FdReport), P]),
        "fd_ddm_solve": (I, [P, P, ctypes.POINTER(P), P, ctypes.POINTER(P), I, D, I, DP, I,
                             ctypes.POINTER(FdReport), P]),
        "fd_arnoldi_step": (I, [I, I, P, P, DP, DP, P]),
        "fd_basis_update": (I, [I, I, P, DP, P, P]),
        "fd_axpby": (I, [I, D, P, D, P, P, P]),
        "fd_norm": (I, [I, P, DP, P]),
        "fd_dot": (I, [I, P, P, DP, P]),
        "fd_comm_unique_id": (I, [ctypes.c_char_p]),
        "fd_comm_init": (I, [ctypes.POINTER(P), I, I, ctypes.c_char_p, I]),
        "fd_comm_init_loopback": (I, [ctypes.POINTER(P), I, I]),
        "fd_comm_rank": (I, [P, ctypes.POINTER(I), ctypes.POINTER(I)]),
        "fd_comm_destroy": (I, [P]),
        "fd_schur_set_comm": (I, [P, P, ctypes.POINTER(I)]),
        "fd_schur_set_stencil": (I, [P, I, I, D, D, D, D, D, D, D, I, I]),
        "fd_ddm_solve_dist": (I, [P, P, ctypes.POINTER(P), P, ctypes.POINTER(P), I, D, I, DP, I,
                                  ctypes.POINTER(FdReport), P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded library; raises NativeError when it has not been built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeError(
                        f"{LIB_PATH} is missing: run `python -m paper_2509_23180_b200.build` "
                        f"(there is no CPU fallback)")
                handle = ctypes.CDLL(LIB_PATH)
                _declare(handle)
                _lib = handle
    return _lib


def check(status: int, report=None):
    if status == FD_OK:
        return
    msg = lib().fd_last_error().decode(errors="replace")
    if status == FD_ERR_VALIDATION:
        raise ValidationError(msg)
    if status == FD_ERR_SINGULAR:
        raise SingularOperatorError(msg)
    if status == FD_ERR_NOT_CONVERGED:
        raise ConvergenceError(msg, report=report)
    if status == FD_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise NativeError(msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


# --- torch buffer helpers -------------------------------------------------------

def torch():
    import torch as _t
    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise NativeError("CUDA device required: the fftddm_b200 path has no CPU fallback")
    lib()


def stream_ptr():
    return P(torch().cuda.current_stream().cuda_stream)


def dptr(x):
    """Device pointer of a contiguous fp64 CUDA tensor."""
    t = torch()
    if not (isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float64 and x.is_contiguous()):
        raise ValidationError("expected a contiguous float64 CUDA tensor")
    return P(x.data_ptr())


def ptr_array(ptrs):
    arr = (P * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p.value if isinstance(p, P) else p
    return arr
