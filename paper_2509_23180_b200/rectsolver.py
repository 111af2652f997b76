"""Single-rectangle fast solver on the GPU (ref fftddm/rectsolver.py).

plan_rect builds a native plan (eigenvalues, compressed per-mode LU factors
and block-carry tables, csrc/plan.cpp); solve_rect runs the fused
DST-I -> Thomas -> DST-I pipeline (csrc/solve.cu).  Scope: the DD transform
along y with ghost-node ends (the reference's default axis choice,
rectsolver.py:24-29,102-109) or along x (the reference's transform_axis "x"
branch, rectsolver.py:111-118,198-199,211-212; also taken when y has no GPU
transform length, see _gpu_axis); the sweep axis may carry any non-periodic
pair with end modifiers (half-cell Dirichlet, Neumann).  Other layouts raise
UnsupportedError.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native, transforms
from ._fields import empty, is_torch, like_input, to_device
from ._native import UnsupportedError
from .errors import SingularOperatorError, ValidationError
from .geometry import BoundaryKind, GridField, RectSubdomain


_PAIR_CODE = {"DD": 0, "NN": 1, "PP": 2}


def _gpu_axis(sub: RectSubdomain) -> str:
    """Transform axis of the GPU plan.  The reference transforms along y when
    that axis is in pure form -- an NN pair, or a DD pair with ghost-node ends
    -- and along x otherwise (rectsolver.py:24-29,102-109); the GPU follows it,
    except that a y length without a GPU transform (n + 1 above 4096 for DD,
    e.g. the c4 south/north arms, n = 16383) moves the transform to a
    transformable x axis (the reference's own transform_axis = "x" branch):
    the FFT stays within one SM's shared memory and the long axis becomes the
    Thomas sweep.  Same operator, rounding-level differences only.  A periodic
    sweep axis (cyclic Thomas) is not on the GPU path."""
    def pair_of(axis):
        try:
            return sub.axis_pair(axis)
        except ValidationError:
            return None

    def ok(axis):
        pair = pair_of(axis)
        if pair in ("NN", "PP"):
            return True
        lo, hi = ("south", "north") if axis == "y" else ("west", "east")
        return pair == "DD" and not sub.end_modifier(lo) and not sub.end_modifier(hi)

    def has_kernel(axis):
        length = sub.n if axis == "y" else sub.m
        return _native.lib().fd_transform_kind_pair(int(length), _PAIR_CODE[pair_of(axis)]) >= 0

    y_ok, x_ok = ok("y"), ok("x")
    if y_ok and (has_kernel("y") or not (x_ok and has_kernel("x"))):
        axis = "y"
    elif x_ok:
        axis = "x"
    else:
        raise UnsupportedError(
            f"subdomain {sub.id}: neither axis is a transformable pair on the GPU path "
            f"(got y {pair_of('y')}, x {pair_of('x')} with end modifiers)")
    sweep = "x" if axis == "y" else "y"
    if pair_of(sweep) == "PP":
        raise UnsupportedError(f"subdomain {sub.id}: periodic sweep axis is not on the GPU path")
    return axis


class _Handle:
    """Owns one native plan handle."""

    def __init__(self, sub: RectSubdomain, axis: str):
        _native.require_cuda()
        h = _native.P()
        pair = _PAIR_CODE[sub.axis_pair(axis)]
        _native.call("fd_plan_create_ex", ctypes_ref(h), sub.m, sub.n, float(sub.dx), float(sub.dy),
                     float(sub.kappa), float(sub.end_modifier("west")), float(sub.end_modifier("east")),
                     float(sub.end_modifier("south")), float(sub.end_modifier("north")),
                     0 if axis == "y" else 1, pair, _native.torch().cuda.current_device())
        self.ptr = h

    def __del__(self):
        try:
            if self.ptr:
                _native.lib().fd_plan_destroy(self.ptr)
        except Exception:
            pass


def ctypes_ref(x):
    import ctypes
    return ctypes.byref(x)


@dataclass(frozen=True)
class RectPlan:
    """Prepared GPU plan for one rectangle (ref rectsolver.py:32-59)."""

    subdomain: RectSubdomain
    transform_axis: str
    y_plan: transforms.SpectralPlan
    solve_pair: str
    off: float
    handle: _Handle = field(repr=False, compare=False)
    pin_mean: bool = False

    @property
    def singular(self) -> bool:
        return False

    @property
    def x_solver_kind(self) -> str:
        return "corner-modified" if self.solve_pair == "NN" else "standard-tridiagonal"

    def info(self) -> dict:
        br, ex, tk = _native.I(), _native.ctypes.c_longlong(), _native.I()
        import ctypes
        _native.call("fd_plan_info", self.handle.ptr, ctypes.byref(br), ctypes.byref(ex),
                     ctypes.byref(tk))
        return {"block_rows": br.value, "explicit_rows": ex.value,
                "transform": ("dense", "fft")[tk.value]}


def plan_rect(subdomain: RectSubdomain, pin_mean: bool = False) -> RectPlan:
    """GPU plan; SingularOperatorError on a zero pivot (ref rectsolver.py:94-180)."""
    sub = subdomain
    if pin_mean:
        raise UnsupportedError("pin_mean (singular all-Neumann operators) is not on the GPU path")
    _native.require_cuda()
    axis = _gpu_axis(sub)
    if axis == "y":
        lam_plan = transforms.make_plan(sub.axis_pair("y"), sub.n, sub.delta_y, sub.delta_x, sub.kappa)
        pair, off = sub.axis_pair("x"), sub.delta_x
    else:
        lam_plan = transforms.make_plan(sub.axis_pair("x"), sub.m, sub.delta_x, sub.delta_y, sub.kappa)
        pair, off = sub.axis_pair("y"), sub.delta_y
    handle = _Handle(sub, axis)
    return RectPlan(subdomain=sub, transform_axis=axis, y_plan=lam_plan,
                    solve_pair=pair, off=off, handle=handle)


def solve_rect(plan: RectPlan, f) -> GridField:
    """A p = f on the rectangle; returns a new GridField (ref rectsolver.py:183-213)."""
    sub = plan.subdomain
    if not isinstance(f, GridField):
        f = GridField(sub.id, f)
    if f.subdomain_id != sub.id:
        raise ValueError(f"field belongs to subdomain {f.subdomain_id}, plan to {sub.id}")
    size = f.values.numel() if is_torch(f.values) else f.values.size
    if size != sub.size:
        raise ValueError(f"field length {size} != {sub.m} x {sub.n}")
    v, host = to_device(f.values, sub.size)
    out = empty(sub.size)
    _native.call("fd_rect_solve", plan.handle.ptr, _native.dptr(v), _native.dptr(out),
                 _native.stream_ptr())
    return GridField(sub.id, like_input(out, host))


def solve_rect_batched(plans, fields, out=None):
    """Solve independent rectangles in one batched launch (torch CUDA tensors
    in and out; this is the config-1 hot path)."""
    fs = [to_device(f.values if isinstance(f, GridField) else f, p.subdomain.size)[0]
          for p, f in zip(plans, fields)]
    outs = out if out is not None else [empty(p.subdomain.size) for p in plans]
    hp = _native.ptr_array([p.handle.ptr for p in plans])
    fp = _native.ptr_array([_native.dptr(f) for f in fs])
    op = _native.ptr_array([_native.dptr(o) for o in outs])
    _native.call("fd_rect_solve_batched", len(plans), hp, fp, op, _native.stream_ptr())
    return outs


def apply_rect_operator(sub: RectSubdomain, values):
    """5-point matvec with end modifiers or periodic wrap (ref rectsolver.py:264-289)."""
    v, host = to_device(values, sub.size)
    out = empty(sub.size)
    ppx, ppy = int(sub.axis_pair("x") == "PP"), int(sub.axis_pair("y") == "PP")
    _native.call("fd_stencil_apply_ex", sub.m, sub.n, float(sub.delta_x), float(sub.delta_y),
                 float(sub.kappa), float(sub.end_modifier("west")), float(sub.end_modifier("east")),
                 float(sub.end_modifier("south")), float(sub.end_modifier("north")), ppx, ppy,
                 _native.dptr(v), _native.dptr(out), _native.stream_ptr())
    return like_input(out, host)


def lift_dirichlet(sub: RectSubdomain, rhs, edge: str, boundary_values):
    """rhs - factor * delta * g on the line next to a Dirichlet edge; factor 2
    for half-cell edges (ref rectsolver.py:292-313).  Host numpy (problem
    assembly) or torch tensors."""
    if sub.edge_bc[edge] is not BoundaryKind.DIRICHLET:
        raise ValueError(f"edge {edge} of subdomain {sub.id} is not Dirichlet")
    factor = 2.0 if edge in sub.half_cell_dirichlet else 1.0
    delta = sub.delta_x if edge in ("west", "east") else sub.delta_y
    if is_torch(rhs):
        G = rhs.reshape(sub.m, sub.n).clone()
        g = _native.torch().as_tensor(boundary_values, dtype=G.dtype, device=G.device)
    else:
        G = np.asarray(rhs, dtype=float).reshape(sub.m, sub.n).copy()
        g = np.asarray(boundary_values, dtype=float)
    sl = {"west": (0, slice(None)), "east": (-1, slice(None)),
          "south": (slice(None), 0), "north": (slice(None), -1)}[edge]
    G[sl] -= factor * delta * g
    return G.reshape(-1)
