"""Device/host field conversion for the drop-in API.

numpy in -> numpy out (one H2D copy in, one D2H copy out); torch CUDA
tensors stay on the device untouched.  This is the only place the package
moves field data between host and device.
"""

from __future__ import annotations

import numpy as np

from ._native import require_cuda, torch
from .errors import ValidationError


def is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def to_device(x, size=None):
    """Flat contiguous fp64 CUDA tensor view/copy of x; returns (tensor, was_numpy)."""
    require_cuda()
    t = torch()
    if is_torch(x):
        v = x.reshape(-1)
        if v.dtype != t.float64:
            v = v.to(t.float64)
        if not v.is_cuda:
            v = v.cuda()
        v = v.contiguous()
        host = False
    else:
        arr = np.ascontiguousarray(np.asarray(x, dtype=float).ravel())
        v = t.from_numpy(arr).cuda()
        host = True
    if size is not None and v.numel() != size:
        raise ValidationError(f"field length {v.numel()} does not match expected size {size}")
    return v, host


def like_input(v, host: bool):
    return v.cpu().numpy() if host else v


def empty(n):
    require_cuda()
    t = torch()
    return t.empty(n, dtype=t.float64, device="cuda")
