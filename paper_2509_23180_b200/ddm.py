"""Schur-complement domain decomposition on the GPU (ref fftddm/ddm.py).

The coupled ("centre") subdomain is eliminated onto its neighbours' fast
solves; the native Schur operator (csrc/driver.cpp) applies
    schur(p)           = sum_i R_ci A_i^{-1} R_ic p         (ddm.py:112-123)
    preconditioned(p)  = p - A_c^{-1} schur(p)              (ddm.py:133-136)
    unpreconditioned(p)= A_c p - schur(p)                   (ddm.py:128-131)
with all neighbour solves batched into one DST/Thomas pipeline launch.
ddm_solve runs Algorithm 1 (ddm.py:210-270) inside the library: arm
pre-solves, reduced right-hand side, GMRES with the basis on the device,
back-substitution.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native, krylov
from ._fields import empty, is_torch, like_input, to_device
from .errors import ConvergenceError, ValidationError
from .geometry import adopt, CompositeDomain, GridField, Interface, line_indices, validate
from .rectsolver import RectPlan, plan_rect, solve_rect


@dataclass(frozen=True)
class CouplingMap:
    """R: `to[to_idx] = coupling * from[from_idx]` (ref ddm.py:27-51)."""

    interface: Interface
    from_id: int
    to_id: int
    from_size: int
    to_size: int
    from_idx: np.ndarray
    to_idx: np.ndarray
    coupling: float

    def apply(self, values):
        shape = tuple(values.shape)
        if shape != (self.from_size,):
            raise ValidationError(f"field length {shape} does not match subdomain "
                                  f"{self.from_id} (size {self.from_size})")
        if is_torch(values):
            t = _native.torch()
            out = t.zeros(self.to_size, dtype=t.float64, device=values.device)
            fi = t.as_tensor(self.from_idx, device=values.device)
            ti = t.as_tensor(self.to_idx, device=values.device)
            out[ti] = self.coupling * values[fi]
            return out
        out = np.zeros(self.to_size)
        out[self.to_idx] = self.coupling * np.asarray(values)[self.from_idx]
        return out


def make_coupling(comp: CompositeDomain, iface: Interface, from_id: int) -> CouplingMap:
    """Coupling map leaving `from_id` across `iface` (ref ddm.py:54-70)."""
    comp, iface = adopt(comp), adopt(iface)
    to_id = iface.other_side(from_id)[0]
    sf, st = comp.subdomain(from_id), comp.subdomain(to_id)
    perm = np.asarray(iface.index_map)
    mine, theirs = (iface.side_a, iface.side_b) if iface.side_a[0] == from_id \
        else (iface.side_b, iface.side_a)
    if mine is iface.side_a:
        fi, ti = line_indices(sf, mine[1]), line_indices(st, theirs[1])[perm]
    else:
        fi, ti = line_indices(sf, mine[1])[perm], line_indices(st, theirs[1])
    return CouplingMap(interface=iface, from_id=from_id, to_id=to_id, from_size=sf.size,
                       to_size=st.size, from_idx=np.asarray(fi, dtype=np.int64),
                       to_idx=np.asarray(ti, dtype=np.int64), coupling=iface.coupling)


def apply_R(cmap: CouplingMap, v: GridField) -> GridField:
    if v.subdomain_id != cmap.from_id:
        raise ValidationError(f"field lives on subdomain {v.subdomain_id}, coupling expects "
                              f"{cmap.from_id}")
    return GridField(cmap.to_id, cmap.apply(v.values))


@dataclass(frozen=True)
class _Neighbor:
    plan: RectPlan
    to_center: CouplingMap      # R_ci
    from_center: CouplingMap    # R_ic
    edge: str = ""              # the neighbour's edge on the interface


def _steklov_line(sub, edge, to_center, from_center):
    """Describe neighbour `sub`'s interface line for the interface-only apply
    (SURVEY 8f row 2), or None when the line is not a ghost-node DD pair.
    Returns (L, M, delta_line, delta_sweep, mod_lo, mod_hi, end, pos_in, pos_out)."""
    if edge in ("west", "east"):
        along, lo, hi, sweep_lo, sweep_hi = "y", "south", "north", "west", "east"
        L, M, dl, ds = sub.n, sub.m, sub.delta_y, sub.delta_x
        pos = lambda idx: np.asarray(idx) % sub.n   # noqa: E731
    else:
        along, lo, hi, sweep_lo, sweep_hi = "x", "west", "east", "south", "north"
        L, M, dl, ds = sub.m, sub.n, sub.delta_x, sub.delta_y
        pos = lambda idx: np.asarray(idx) // sub.n  # noqa: E731
    try:
        if sub.axis_pair(along) != "DD" or sub.end_modifier(lo) or sub.end_modifier(hi):
            return None
        if sub.axis_pair("x" if along == "y" else "y") == "PP":
            return None
    except ValidationError:
        return None
    end = 0 if edge in ("west", "south") else 1
    return (L, M, dl, ds, float(sub.end_modifier(sweep_lo)), float(sub.end_modifier(sweep_hi)), end,
            np.ascontiguousarray(pos(from_center.to_idx), dtype=np.int64),
            np.ascontiguousarray(pos(to_center.from_idx), dtype=np.int64))


class _SchurHandle:
    def __init__(self, center_plan, neighbors):
        c = center_plan.subdomain
        nb = len(neighbors)
        h = _native.P()
        plans = _native.ptr_array([n.plan.handle.ptr for n in neighbors])
        lens = (ctypes.c_int * max(nb, 1))(*[len(n.to_center.from_idx) for n in neighbors])
        keep = []

        def arr(xs):
            a = (ctypes.c_void_p * max(nb, 1))()
            for i, x in enumerate(xs):
                x = np.ascontiguousarray(x, dtype=np.int64)
                keep.append(x)
                a[i] = x.ctypes.data
            return a

        def dbl(xs):
            return (ctypes.c_double * max(nb, 1))(*[float(x) for x in xs])

        _native.call("fd_schur_create", ctypes.byref(h), center_plan.handle.ptr,
                     float(c.end_modifier("south")), float(c.end_modifier("north")), nb, plans, lens,
                     arr([n.to_center.from_idx for n in neighbors]),
                     arr([n.to_center.to_idx for n in neighbors]),
                     dbl([n.to_center.coupling for n in neighbors]),
                     arr([n.from_center.from_idx for n in neighbors]),
                     arr([n.from_center.to_idx for n in neighbors]),
                     dbl([n.from_center.coupling for n in neighbors]))
        self.ptr = h

    def __del__(self):
        try:
            if self.ptr:
                _native.lib().fd_schur_destroy(self.ptr)
        except Exception:
            pass

    def use_interface_only(self, neighbors, kappa) -> bool:
        """Switch the neighbour applies to the interface-only (Steklov) form when
        every neighbour's interface line qualifies; returns whether it did."""
        lines = [_steklov_line(nb.plan.subdomain, nb.edge, nb.to_center, nb.from_center) for nb in neighbors]
        if not lines or any(x is None for x in lines) or len({x[0] for x in lines}) != 1:
            return False
        for i, (L, M, dl, ds, mlo, mhi, end, pin, pout) in enumerate(lines):
            st = _native.lib().fd_schur_set_steklov(self.ptr, i, L, M, float(dl), float(ds), float(kappa),
                                                    mlo, mhi, end, pin.ctypes.data, pout.ctypes.data)
            if st == _native.FD_ERR_UNSUPPORTED:
                return False
            _native.check(st)
        _native.call("fd_schur_use_steklov", self.ptr, 1)
        return True


@dataclass(frozen=True)
class SchurOperator:
    """Matrix-free (A_c - sum S) on the coupled subdomain (ref ddm.py:94-136).
    Methods take numpy or torch CUDA vectors and return the same kind."""

    coupled_id: int
    center: object
    center_plan: RectPlan
    neighbors: tuple
    handle: _SchurHandle
    pool: object = None

    @property
    def size(self) -> int:
        return self.center.size

    def _run(self, name, p):
        v, host = to_device(p, self.size)
        out = empty(self.size)
        _native.call(name, self.handle.ptr, _native.dptr(v), _native.dptr(out), _native.stream_ptr())
        return like_input(out, host)

    def schur(self, p):
        return self._run("fd_schur_apply", p)

    def center_solve(self, rhs):
        return self._run("fd_center_solve", rhs)

    def preconditioned(self, p):
        return self._run("fd_precond_apply", p)

    def unpreconditioned(self, p):
        return self._run("fd_unprecond_apply", p)


def apply_schur(op: SchurOperator, p: GridField) -> GridField:
    if p.subdomain_id != op.coupled_id:
        raise ValidationError("field is not on the coupled subdomain")
    return GridField(op.coupled_id, op.schur(p.values))


def apply_preconditioned_operator(op: SchurOperator, p: GridField) -> GridField:
    if p.subdomain_id != op.coupled_id:
        raise ValidationError("field is not on the coupled subdomain")
    return GridField(op.coupled_id, op.preconditioned(p.values))


def solver_threads() -> int:
    """SOLVER_THREADS semantics kept for API compatibility (ref ddm.py:152-163);
    the GPU path batches neighbour solves instead of using host threads."""
    raw = os.environ.get("SOLVER_THREADS", "")
    if not raw.strip():
        return os.cpu_count() or 1
    try:
        count = int(raw)
    except ValueError:
        raise ValidationError(f"SOLVER_THREADS must be an integer, got {raw!r}") from None
    if count < 1:
        raise ValidationError(f"SOLVER_THREADS must be positive, got {count}")
    return count


def designate_center(comp: CompositeDomain) -> int:
    """The unique subdomain with >= 2 interfaces, else the lowest id (ref ddm.py:166-179)."""
    coupled = sorted(comp.coupled_ids)
    if len(coupled) > 1:
        raise ValidationError(f"more than one coupled subdomain: {coupled}")
    if coupled:
        return coupled[0]
    if not comp.interfaces:
        raise ValidationError("composite has no interfaces")
    return min(s.id for s in comp.subdomains)


def build_schur_operator(comp: CompositeDomain, coupled_id: int | None = None,
                         threads: int | None = None, interface_only: bool = False) -> SchurOperator:
    """Plans for the centre and every neighbour + native operator (ref ddm.py:182-201).
    interface_only=True selects the opt-in Steklov form of the neighbour applies
    (same operator up to rounding) when every neighbour's
    interface line is a ghost-node DD pair of one length."""
    comp = adopt(comp)
    if coupled_id is None:
        coupled_id = designate_center(comp)
    center = comp.subdomain(coupled_id)
    neighbors = []
    for iface in comp.interfaces_of(coupled_id):
        other = iface.other_side(coupled_id)[0]
        edge = iface.side_a[1] if iface.side_a[0] == other else iface.side_b[1]
        neighbors.append(_Neighbor(plan=plan_rect(comp.subdomain(other)),
                                   to_center=make_coupling(comp, iface, other),
                                   from_center=make_coupling(comp, iface, coupled_id), edge=edge))
    cplan = plan_rect(center)
    handle = _SchurHandle(cplan, neighbors)
    # A_c in the caller's layout (periodic axes, transposed plans): rectsolver.py:264-289
    _native.call("fd_schur_set_stencil", handle.ptr, center.m, center.n, float(center.delta_x),
                 float(center.delta_y), float(center.kappa), float(center.end_modifier("west")),
                 float(center.end_modifier("east")), float(center.end_modifier("south")),
                 float(center.end_modifier("north")), int(center.axis_pair("x") == "PP"),
                 int(center.axis_pair("y") == "PP"))
    if interface_only:
        kappas = {comp.subdomain(nb.plan.subdomain.id).kappa for nb in neighbors}
        if len(kappas) == 1:
            handle.use_interface_only(neighbors, kappas.pop())
    return SchurOperator(coupled_id=coupled_id, center=center, center_plan=cplan,
                         neighbors=tuple(neighbors), handle=handle)


def ddm_solve(comp: CompositeDomain, f, gmres_cfg=None, coupled_id: int | None = None,
              interface_only: bool = False):
    """Solve the composite system; returns ({id: GridField}, SolveReport)
    (ref ddm.py:210-270).  numpy right-hand sides give numpy solutions; torch
    CUDA right-hand sides stay on the device."""
    comp = adopt(comp)
    validate(comp).require()
    cfg = gmres_cfg or krylov.GmresConfig()
    rhs, host = {}, True
    for sub in comp.subdomains:
        fi = f[sub.id]
        vals = fi.values if isinstance(fi, GridField) else fi
        n = vals.numel() if is_torch(vals) else np.asarray(vals).size
        if n != sub.size or (not is_torch(vals) and np.asarray(vals).ndim != 1):
            raise ValidationError(f"rhs for subdomain {sub.id} has length {n}, expected {sub.size}")
        rhs[sub.id], host = to_device(vals, sub.size)
    if not comp.interfaces:
        (sub,) = comp.subdomains
        p = solve_rect(plan_rect(sub), rhs[sub.id])
        rep = krylov.SolveReport(True, 0, np.zeros(1), 0.0)
        return {sub.id: GridField(sub.id, like_input(p.values, host))}, rep
    if cfg.preconditioner != "fft":
        return _ddm_solve_generic(comp, rhs, cfg, coupled_id, host)
    op = build_schur_operator(comp, coupled_id=coupled_id, interface_only=interface_only)
    nbs = [nb.plan.subdomain for nb in op.neighbors]
    p_c = empty(op.size)
    p_nb = [empty(s.size) for s in nbs]
    hist = np.zeros(cfg.m * cfg.max_restarts + 2)
    rep = _native.FdReport()
    st = _native.lib().fd_ddm_solve(
        op.handle.ptr, _native.dptr(rhs[op.coupled_id]),
        _native.ptr_array([_native.dptr(rhs[s.id]) for s in nbs]), _native.dptr(p_c),
        _native.ptr_array([_native.dptr(x) for x in p_nb]), cfg.m, cfg.tol, cfg.max_restarts,
        hist.ctypes.data_as(_native.DP), hist.size, ctypes.byref(rep), _native.stream_ptr())
    report = krylov.report_from_native(rep, hist)
    fields = {op.coupled_id: GridField(op.coupled_id, like_input(p_c, host))}
    for s, x in zip(nbs, p_nb):
        fields[s.id] = GridField(s.id, like_input(x, host))
    if st == _native.FD_ERR_NOT_CONVERGED:
        err = ConvergenceError(_native.lib().fd_last_error().decode(), report=report)
        err.solution = fields[op.coupled_id].values
        raise err
    _native.check(st)
    return fields, report


def _ddm_solve_generic(comp, rhs, cfg, coupled_id, host):
    """identity / jacobi preconditioners (comparison studies, ref krylov.py:179-186)
    through the same native operator applies, GMRES driven from Python."""
    op = build_schur_operator(comp, coupled_id=coupled_id)
    arms = list(op.neighbors)
    qs = [solve_rect(nb.plan, rhs[nb.plan.subdomain.id]).values for nb in arms]
    fp = rhs[op.coupled_id].clone()
    for nb, q in zip(arms, qs):
        fp -= nb.to_center.apply(q)
    p_c, report = krylov.solve_coupled(op, GridField(op.coupled_id, fp), cfg)
    fields = {op.coupled_id: GridField(op.coupled_id, like_input(p_c.values, host))}
    for nb, q in zip(arms, qs):
        corr = solve_rect(nb.plan, nb.from_center.apply(p_c.values)).values
        sid = nb.plan.subdomain.id
        fields[sid] = GridField(sid, like_input(q - corr, host))
    return fields, report
