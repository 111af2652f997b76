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

The local arithmetic is a pluggable backend: `GpuBackend` (production:
native plans/solves, device GMRES with native Arnoldi kernels) or any object
with the same methods (tests/test_dist_gloo.py drives the protocol on CPU
with the oracle).
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
