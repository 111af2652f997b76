"""Device/host field conversion for the drop-in API.

numpy in -> numpy out (one H2D copy in, one D2H copy out); torch CUDA
tensors stay on the device untouched.  This is the only place the package
moves field data between host and device.

Host data goes through page-locked memory: inputs are copied into a pinned
staging buffer (reused between calls) and sent with one asynchronous DMA on
the current stream; outputs are read back by one DMA into page-locked arrays
that the caller receives as numpy views (no second host copy).
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
        arr = np.asarray(x, dtype=float).ravel()
        stage = _staging(arr.size)
        np.copyto(stage.numpy(), arr)
        v = t.empty(arr.size, dtype=t.float64, device="cuda")
        v.copy_(stage, non_blocking=True)
        _in_flight.append((stage, t.cuda.current_stream().record_event()))
        host = True
    if size is not None and v.numel() != size:
        raise ValidationError(f"field length {v.numel()} does not match expected size {size}")
    return v, host


# pinned staging buffers of the inputs: reused once the copy that read one has
# completed (event), so back-to-back calls do not allocate page-locked memory
_free_stage: list = []
_in_flight: list = []


def _staging(n):
    t = torch()
    keep = []
    for stage, ev in _in_flight:
        if ev.query():
            _free_stage.append(stage)
        else:
            keep.append((stage, ev))
    _in_flight[:] = keep
    for i, buf in enumerate(_free_stage):
        if buf.numel() >= n:
            return _free_stage.pop(i)[:n]
    return t.empty(n, dtype=t.float64, pin_memory=True)


def like_input(v, host: bool):
    """Device field back to the caller's kind: numpy (pinned, one DMA) or torch."""
    if not host:
        return v
    t = torch()
    out = t.empty(v.numel(), dtype=t.float64, pin_memory=True)
    out.copy_(v.reshape(-1), non_blocking=True)
    t.cuda.current_stream().synchronize()
    return out.numpy()


def empty(n):
    require_cuda()
    t = torch()
    return t.empty(n, dtype=t.float64, device="cuda")
