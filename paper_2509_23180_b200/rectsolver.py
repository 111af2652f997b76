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
from .geometry import adopt, BoundaryKind, GridField, RectSubdomain


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
    sweep axis runs the cyclic (Sherman-Morrison) solve on the dense path."""
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

    # kernel ranking: the fused FFT solve, then the dense-table solve, then the
    # any-length (Stockham / Bluestein) passes; none
    rank_of = {1: 3, 0: 2, 2: 1}

    def rank(axis):
        length = sub.n if axis == "y" else sub.m
        return rank_of.get(_native.lib().fd_transform_kind_pair(int(length), _PAIR_CODE[pair_of(axis)]), 0)

    y_ok, x_ok = ok("y"), ok("x")
    # the reference prefers y (rectsolver.py:102-109); x only for a strictly faster kernel
    if y_ok and (not x_ok or rank("y") >= rank("x")):
        axis = "y"
    elif x_ok:
        axis = "x"
    else:
        raise UnsupportedError(
            f"subdomain {sub.id}: neither axis is a transformable pair on the GPU path "
            f"(got y {pair_of('y')}, x {pair_of('x')} with end modifiers)")
    return axis


class _Handle:
    """Owns one native plan handle."""

    def __init__(self, sub: RectSubdomain, axis: str, cyclic: bool = False, pin_mean: bool = False):
        _native.require_cuda()
        h = _native.P()
        pair = _PAIR_CODE[sub.axis_pair(axis)]
        _native.call("fd_plan_create_sweep", ctypes_ref(h), sub.m, sub.n, float(sub.dx), float(sub.dy),
                     float(sub.kappa), float(sub.end_modifier("west")), float(sub.end_modifier("east")),
                     float(sub.end_modifier("south")), float(sub.end_modifier("north")),
                     0 if axis == "y" else 1, pair, int(cyclic), int(pin_mean),
                     _native.torch().cuda.current_device())
        self.ptr = h

    def singular_modes(self) -> tuple:
        import ctypes
        cnt = _native.I()
        _native.call("fd_plan_singular_modes", self.ptr, None, 0, ctypes.byref(cnt))
        if not cnt.value:
            return ()
        buf = (_native.I * cnt.value)()
        _native.call("fd_plan_singular_modes", self.ptr, buf, cnt.value, ctypes.byref(cnt))
        return tuple(int(v) for v in buf)

    def set_pinv(self, mats) -> None:
        import ctypes
        arr = np.ascontiguousarray(np.stack(mats), dtype=np.float64)
        _native.call("fd_plan_set_pinv", self.ptr, len(mats),
                     arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))

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
    cyclic: bool = False
    singular_modes: tuple = ()

    @property
    def singular(self) -> bool:
        return bool(self.singular_modes)

    @property
    def x_solver_kind(self) -> str:
        if self.cyclic:
            return "cyclic"
        return "corner-modified" if self.solve_pair == "NN" else "standard-tridiagonal"

    def info(self) -> dict:
        br, ex, tk = _native.I(), _native.ctypes.c_longlong(), _native.I()
        import ctypes
        _native.call("fd_plan_info", self.handle.ptr, ctypes.byref(br), ctypes.byref(ex),
                     ctypes.byref(tk))
        return {"block_rows": br.value, "explicit_rows": ex.value,
                "transform": ("dense", "fft", "sep")[tk.value]}


def _sweep_matrix(lam_k: float, ms: int, off: float, cyclic: bool, mod_lo: float, mod_hi: float):
    """Dense per-mode sweep matrix of a singular mode (rectsolver.py:164-173)."""
    d = np.full(ms, lam_k)
    if not cyclic:
        d[0] += mod_lo
        d[-1] += mod_hi
    M = np.diag(d)
    idx = np.arange(ms - 1)
    M[idx, idx + 1] += off
    M[idx + 1, idx] += off
    if cyclic:
        M[0, ms - 1] += off
        M[ms - 1, 0] += off
    return M


def plan_rect(subdomain: RectSubdomain, pin_mean: bool = False) -> RectPlan:
    """GPU plan (ref rectsolver.py:94-180).  SingularOperatorError on a zero
    pivot unless pin_mean is set; then the singular modes are solved in the
    minimum-norm sense: their sweep matrices' pseudo-inverses are formed here
    at plan time (host setup, like the reference's dense mode matrices) and
    applied on the device inside the solve."""
    subdomain = adopt(subdomain)
    sub = subdomain
    _native.require_cuda()
    axis = _gpu_axis(sub)
    if axis == "y":
        lam_plan = transforms.make_plan(sub.axis_pair("y"), sub.n, sub.delta_y, sub.delta_x, sub.kappa)
        pair, off, ms, lo, hi = sub.axis_pair("x"), sub.delta_x, sub.m, "west", "east"
    else:
        lam_plan = transforms.make_plan(sub.axis_pair("x"), sub.m, sub.delta_x, sub.delta_y, sub.kappa)
        pair, off, ms, lo, hi = sub.axis_pair("y"), sub.delta_y, sub.n, "south", "north"
    cyclic = pair == "PP"
    if cyclic and ms % 2:
        raise ValidationError(f"subdomain {sub.id}: periodic sweep axis needs an even count")
    handle = _Handle(sub, axis, cyclic=cyclic, pin_mean=pin_mean)
    singular = handle.singular_modes() if pin_mean else ()
    if singular:
        lam = np.asarray(lam_plan.eigenvalues)
        mats = []
        for k in singular:
            M = _sweep_matrix(lam[k], ms, off, cyclic, sub.end_modifier(lo), sub.end_modifier(hi))
            # lstsq(M, f, rcond=None) == pinv(M) f with the same cutoff (rectsolver.py:207)
            mats.append(np.linalg.pinv(M, rcond=np.finfo(float).eps * ms))
        handle.set_pinv(mats)
    return RectPlan(subdomain=sub, transform_axis=axis, y_plan=lam_plan,
                    solve_pair=pair, off=off, handle=handle, pin_mean=pin_mean,
                    cyclic=cyclic, singular_modes=tuple(singular))


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
    sub = adopt(sub)
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
    sub = adopt(sub)
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
