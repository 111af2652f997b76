"""Subdomain-sharded Algorithm 1 over torch.distributed.

Rank 0 owns the coupled (centre) subdomain, runs GMRES and keeps the Krylov
basis; the neighbour ("arm") subdomains are dealt round-robin to ranks
1..W-1 (to rank 0 when W == 1).  One operator application (ddm.py:133-136):

    rank 0  --R_ic line (<= n doubles)-->  arm owner   (send)
    arm owner: g = 0 + line, q = A_i^{-1} g              (local fast solve)
    arm owner --R_ci line-->  rank 0                     (send)
    rank 0: s = sum of lines (neighbour order), p - A_c^{-1} s

All arm solves of one application run concurrently on their ranks; messages
are tiny (one interface line, <= 32 KB at n = 4095) and point-to-point
(NCCL send/recv over NVLink on GPUs, gloo on CPU).  The pre-solves, the
reduced right-hand side f' (ddm.py:249-254) and the back-substitution
(ddm.py:259-269) follow the same pattern.  The arithmetic of each piece is
the single-GPU path's; only where it runs changes, so results equal the
single-process solve to rounding.

The local arithmetic is a pluggable backend: `GpuBackend` (native plans and
solves, GMRES driven from Python) or any object with the same methods
(tests/test_dist_gloo.py drives the protocol on CPU with the oracle).

`sharded_ddm_solve` is the production path: the same protocol inside the
native library (fd_ddm_solve_dist: NCCL point-to-point on the caller's
stream, the low-synchronisation device GMRES on rank 0, no Python in the
loop), with a communicator from `nccl_comm` (one process per GPU, the NCCL id
broadcast over torch.distributed) or `loopback_comms` (in-process ranks on one
device: the test transport).
"""

from __future__ import annotations

import numpy as np

from .errors import ValidationError
from .geometry import validate

CMD_DONE, CMD_APPLY, CMD_BACKSUB = 0, 1, 2


class GpuBackend:
    """Local arithmetic on this rank's GPU through the native library."""

    def __init__(self):
        import torch

        from . import _native
        _native.require_cuda()
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device())

    def plan(self, sub):
        from .rectsolver import plan_rect
        return plan_rect(sub)

    def solve(self, plan, v):
        from .rectsolver import solve_rect
        return solve_rect(plan, v).values

    def array(self, x):
        return self.torch.as_tensor(np.asarray(x) if not hasattr(x, "device") else x,
                                    dtype=self.torch.float64, device=self.dev).reshape(-1)

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.dev)

    def index(self, idx):
        return self.torch.as_tensor(np.asarray(idx), device=self.dev)

    # message buffers: device tensors for NCCL; host tensors when the process
    # group is gloo (functional runs without NCCL)
    host_comm = False

    def comm(self, x):
        return x.detach().cpu().contiguous() if self.host_comm else x.contiguous()

    def empty_comm(self, n):
        return self.torch.empty(n, dtype=self.torch.float64, device="cpu" if self.host_comm else self.dev)

    def from_comm(self, t):
        return t.to(self.dev) if self.host_comm else t

    def gmres(self, op, rhs, cfg):
        from .krylov import gmres
        return gmres(op, rhs, cfg=cfg)

    def norm(self, v):
        return float(self.torch.linalg.norm(v))

    def stencil(self, sub, v):
        from .rectsolver import apply_rect_operator
        return apply_rect_operator(sub, v)


def owners(n_arms: int, world: int):
    """Rank owning arm i: round-robin over ranks 1..W-1 (rank 0 if alone)."""
    if world <= 1:
        return [0] * n_arms
    return [1 + (i % (world - 1)) for i in range(n_arms)]


def dist_ddm_solve(comp, f, gmres_cfg=None, coupled_id=None, backend=None, group=None):
    """Distributed ddm_solve.  Every rank passes the same composite and the
    right-hand sides of (at least) the subdomains it owns.  Returns
    ({sid: field} for the subdomains this rank owns, SolveReport on rank 0 /
    None elsewhere)."""
    import torch.distributed as dist

    from . import krylov
    from .ddm import designate_center, make_coupling

    validate(comp).require()
    cfg = gmres_cfg or krylov.GmresConfig()
    be = backend or GpuBackend()
    if isinstance(be, GpuBackend) and dist.is_initialized():
        be.host_comm = dist.get_backend(group) == "gloo"
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if coupled_id is None:
        coupled_id = designate_center(comp)
    center = comp.subdomain(coupled_id)
    arms = []
    for iface in comp.interfaces_of(coupled_id):
        other = iface.other_side(coupled_id)[0]
        arms.append((comp.subdomain(other), make_coupling(comp, iface, other),
                     make_coupling(comp, iface, coupled_id)))
    own = owners(len(arms), world)

    def send(t, dst):
        dist.send(be.comm(t), dst, group=group)

    def recv(n, src):
        buf = be.empty_comm(n)
        dist.recv(buf, src, group=group)
        return be.from_comm(buf)

    # ---------------- arm owners (incl. rank 0 when it owns arms) ----------------
    local = {}
    for i, (sub, to_c, from_c) in enumerate(arms):
        if own[i] == rank:
            fi = f[sub.id]
            fi = fi.values if hasattr(fi, "values") else fi
            pl = be.plan(sub)
            q = be.solve(pl, be.array(fi))                       # pre-solve (ddm.py:249-250)
            local[i] = {"sub": sub, "plan": pl, "q": q, "to_c": to_c, "from_c": from_c,
                        "to_from": be.index(to_c.from_idx), "from_to": be.index(from_c.to_idx)}

    def arm_apply(i, line):
        """q = A_i^{-1} (R_ic p) given the raw centre line p[from_idx]; returns
        (q, R_ci q restricted to the centre line)."""
        a = local[i]
        g = be.zeros(a["sub"].size)
        g[a["from_to"]] = a["from_c"].coupling * line
        q = be.solve(a["plan"], g)
        return q, a["to_c"].coupling * q[a["to_from"]]

    if rank != 0 and not local:
        return {}, None                                        # no arm here: nothing to serve
    if rank != 0:
        # pre-solve lines to rank 0, then serve operator applications
        for i in sorted(local):
            send(local[i]["to_c"].coupling * local[i]["q"][local[i]["to_from"]], 0)
        out = {}
        while True:
            cmd = int(recv(1, 0)[0].item())
            if cmd == CMD_DONE:
                break
            # receive every line first, then reply: no send waits on a pending send
            lines = {i: recv(len(local[i]["from_c"].from_idx), 0) for i in sorted(local)}
            for i in sorted(local):
                q, back = arm_apply(i, lines[i])
                if cmd == CMD_APPLY:
                    send(back, 0)
                else:                                          # back-substitution
                    out[local[i]["sub"].id] = local[i]["q"] - q
        return out, None

    # ---------------- rank 0: centre, GMRES, protocol driver ----------------
    cplan = be.plan(center)
    c_from = [be.index(fc.from_idx) for _, _, fc in arms]      # centre indices of R_ic
    c_to = [be.index(tc.to_idx) for _, tc, _ in arms]          # centre indices of R_ci
    lines_in = [None] * len(arms)
    for i in range(len(arms)):
        if own[i] == 0:
            a = local[i]
            lines_in[i] = a["to_c"].coupling * a["q"][a["to_from"]]
    for r in range(1, world):
        for i in range(len(arms)):
            if own[i] == r:
                lines_in[i] = recv(len(arms[i][1].from_idx), r)
    fc = f[coupled_id]
    fc = be.array(fc.values if hasattr(fc, "values") else fc)
    f_prime = fc.clone() if hasattr(fc, "clone") else fc.copy()
    for i in range(len(arms)):                                 # f' = f_c - sum R_ci q_i
        f_prime[c_to[i]] = f_prime[c_to[i]] - lines_in[i]

    def broadcast_lines(cmd, p):
        for r in range(1, world):
            if any(o == r for o in own):
                send(be.array([float(cmd)]), r)
        for r in range(1, world):
            for i in range(len(arms)):
                if own[i] == r:
                    send(p[c_from[i]], r)

    def schur(p):
        broadcast_lines(CMD_APPLY, p)
        backs = [None] * len(arms)
        for i in range(len(arms)):
            if own[i] == 0:
                backs[i] = arm_apply(i, p[c_from[i]])[1]
        for r in range(1, world):
            for i in range(len(arms)):
                if own[i] == r:
                    backs[i] = recv(len(arms[i][1].from_idx), r)
        s = be.zeros(center.size)
        for i in range(len(arms)):                             # out += part, neighbour order
            s[c_to[i]] = s[c_to[i]] + backs[i]
        return s

    def preconditioned(p):
        return p - be.solve(cplan, schur(p))

    # every serving rank always gets CMD_DONE, also when GMRES raises
    # (ConvergenceError) or anything else fails on rank 0
    try:
        rhs = be.solve(cplan, f_prime)                         # krylov.py:178
        x, report = be.gmres(preconditioned, rhs, cfg)
        resid = be.stencil(center, x) - schur(x) - f_prime     # krylov.py:189
        report = krylov.SolveReport(report.converged, report.iterations, report.residual_history,
                                    report.wall_time, be.norm(resid))
        # back-substitution p_i = q_i - A_i^{-1} R_ic p_c
        broadcast_lines(CMD_BACKSUB, x)
        out = {coupled_id: x}
        for i in range(len(arms)):
            if own[i] == 0:
                q, _ = arm_apply(i, x[c_from[i]])
                out[local[i]["sub"].id] = local[i]["q"] - q
    finally:
        for r in range(1, world):
            if any(o == r for o in own):
                send(be.array([float(CMD_DONE)]), r)
    return out, report


def check_world(comp, world):
    n_arms = max(len(comp.interfaces_of(s.id)) for s in comp.subdomains)
    if world > n_arms + 1:
        raise ValidationError(f"{world} ranks for {n_arms} arms: extra ranks would idle")


# ---------------------------------------------------------------------------
# native sharded solve (fd_ddm_solve_dist)

class Comm:
    """Owns one native communicator handle (fd_comm)."""

    def __init__(self, ptr, rank, world):
        self.ptr, self.rank, self.world = ptr, rank, world

    def __del__(self):
        try:
            if self.ptr:
                from . import _native
                _native.lib().fd_comm_destroy(self.ptr)
        except Exception:
            pass


def nccl_comm(group=None):
    """NCCL communicator over the torch.distributed process group: rank 0
    draws the NCCL unique id, every rank receives it by broadcast."""
    import ctypes

    import torch
    import torch.distributed as dist

    from . import _native
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ident = ctypes.create_string_buffer(128)
    if rank == 0:
        _native.call("fd_comm_unique_id", ident)
    obj = [bytes(ident.raw)]
    dist.broadcast_object_list(obj, src=0, group=group)
    h = _native.P()
    _native.call("fd_comm_init", ctypes.byref(h), world, rank, obj[0], torch.cuda.current_device())
    return Comm(h, rank, world)


def loopback_comms(world: int):
    """`world` in-process ranks on the current device (the protocol's test
    transport: host-side hand-off, no kernel waits on another rank)."""
    import ctypes

    import torch

    from . import _native
    arr = (_native.P * world)()
    _native.call("fd_comm_init_loopback", arr, world, torch.cuda.current_device())
    return [Comm(_native.P(arr[r]), r, world) for r in range(world)]


def sharded_ddm_solve(comp, f, comm: Comm, gmres_cfg=None, coupled_id=None, owner=None):
    """Algorithm 1 sharded over `comm`'s ranks inside the native library.  Every
    rank passes the same composite and the right-hand sides of the subdomains
    it owns (rank 0: the centre; arms: `owners`).  Returns ({sid: field} of the
    owned subdomains, SolveReport on rank 0 / None elsewhere)."""
    import ctypes

    import numpy as np

    from . import _native, krylov
    from ._fields import empty, to_device
    from .ddm import build_schur_operator
    from .errors import ConvergenceError
    from .geometry import GridField

    validate(comp).require()
    cfg = gmres_cfg or krylov.GmresConfig()
    op = build_schur_operator(comp, coupled_id=coupled_id)
    nbs = [nb.plan.subdomain for nb in op.neighbors]
    own = list(owner) if owner is not None else owners(len(nbs), comm.world)
    _native.call("fd_schur_set_comm", op.handle.ptr, comm.ptr, (ctypes.c_int * max(len(own), 1))(*own))
    mine = [own[i] == comm.rank for i in range(len(nbs))]
    rhs = {}
    for i, s_ in enumerate(nbs):
        if mine[i]:
            fi = f[s_.id]
            rhs[s_.id] = to_device(fi.values if isinstance(fi, GridField) else fi, s_.size)[0]
    p_nb = [empty(s_.size) if mine[i] else None for i, s_ in enumerate(nbs)]
    f_nb = _native.ptr_array([_native.dptr(rhs[s_.id]) if mine[i] else 0 for i, s_ in enumerate(nbs)])
    pp_nb = _native.ptr_array([_native.dptr(x) if x is not None else 0 for x in p_nb])
    hist = np.zeros(cfg.m * cfg.max_restarts + 2)
    rep = _native.FdReport()
    fc = pc = None
    if comm.rank == 0:
        fi = f[op.coupled_id]
        fc = to_device(fi.values if isinstance(fi, GridField) else fi, op.size)[0]
        pc = empty(op.size)
    st = _native.lib().fd_ddm_solve_dist(
        op.handle.ptr, _native.dptr(fc) if fc is not None else None, f_nb,
        _native.dptr(pc) if pc is not None else None, pp_nb, cfg.m, cfg.tol, cfg.max_restarts,
        hist.ctypes.data_as(_native.DP), hist.size, ctypes.byref(rep), _native.stream_ptr())
    fields = {s_.id: GridField(s_.id, x) for s_, x in zip(nbs, p_nb) if x is not None}
    report = None
    if comm.rank == 0:
        fields[op.coupled_id] = GridField(op.coupled_id, pc)
        report = krylov.report_from_native(rep, hist)
        if st == _native.FD_ERR_NOT_CONVERGED:
            err = ConvergenceError(_native.lib().fd_last_error().decode(), report=report)
            err.solution = pc
            raise err
    _native.check(st)
    return fields, report
