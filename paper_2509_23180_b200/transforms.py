"""Eigenbasis transforms of the 1-D axis operators (ref fftddm/transforms.py).

`eigenvalues`/`make_plan` are host-side setup (O(n)).  `apply_Q`/`apply_Qt`
run on torch CUDA tensors (numpy input is copied to the device and the result
back) for every length: the DD pair (Q = Q^T = sqrt(2/(n+1)) DST-I,
transforms.py:112-113,135-136) on the real-symmetric FFT kernel when n + 1 is
a power of two in [256, 4096], on the dense periodic-table transform for
n <= 2048, otherwise on the any-length passes (power-of-two Stockham or
Bluestein, csrc/fft_any.cu); NN (DCT-II/III) and PP (real Fourier, even n)
likewise (dense table up to 2048, any-length passes above).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from ._fields import is_torch, require_cuda
from ._native import UnsupportedError

BC_PAIRS = ("DD", "NN", "PP")


def eigenvalues(bc: str, n: int, delta_t: float, delta_o: float, kappa: float = 0.0) -> np.ndarray:
    """Eigenvalues ordered like apply_Q's basis (ref transforms.py:26-38)."""
    j = np.arange(1, n + 1, dtype=float)
    if bc == "DD":
        cosarg = np.cos(j * np.pi / (n + 1))
    elif bc == "NN":
        cosarg = np.cos((j - 1) * np.pi / n)
    elif bc == "PP":
        cosarg = np.cos(2.0 * np.pi * (j - 1) / n)
    else:
        raise ValueError(f"unknown BC pair {bc!r}")
    return -2.0 * (delta_t + delta_o) + 2.0 * delta_t * cosarg + kappa


@dataclass(frozen=True)
class SpectralPlan:
    bc: str
    n: int
    delta_t: float
    delta_o: float
    kappa: float
    eigenvalues: np.ndarray


def make_plan(bc: str, n: int, delta_t: float, delta_o: float, kappa: float = 0.0) -> SpectralPlan:
    if n < 1:
        raise ValueError("transform length must be >= 1")
    if bc not in BC_PAIRS:
        raise ValueError(f"unknown BC pair {bc!r}")
    if bc == "PP" and n % 2:
        raise ValueError("periodic transforms need an even length")
    lam = eigenvalues(bc, n, delta_t, delta_o, kappa)
    lam.setflags(write=False)
    return SpectralPlan(bc, n, delta_t, delta_o, kappa, lam)


_PAIR = {"DD": 0, "NN": 1, "PP": 2}


def _apply(plan: SpectralPlan, v, inverse: bool):
    require_cuda()
    t = _native.torch()
    host = not is_torch(v)
    x = t.as_tensor(np.asarray(v, dtype=float)) if host else v
    if x.shape[-1] != plan.n:
        raise ValueError(f"length mismatch: expected {plan.n}, got {x.shape[-1]}")
    shape = x.shape
    rows = x.reshape(-1, plan.n).to(device="cuda", dtype=t.float64).contiguous()
    out = t.empty_like(rows)
    _native.call("fd_transform_rows", rows.shape[0], plan.n, _PAIR[plan.bc], int(inverse),
                 _native.dptr(rows), _native.dptr(out), t.cuda.current_device(), _native.stream_ptr())
    out = out.reshape(shape)
    return out.cpu().numpy() if host else out


def apply_Q(plan: SpectralPlan, v):
    """Q @ v along the last axis (ref transforms.py:106-126)."""
    return _apply(plan, v, True)


def apply_Qt(plan: SpectralPlan, v):
    """Q^T @ v along the last axis; Q is symmetric for DD (ref transforms.py:129-148)."""
    return _apply(plan, v, False)
