"""Problem builders for BASELINE.json configs c0-c4.

Every builder is written against a *geometry API namespace* so the same
recipe drives both this package and the reference (`api=fftddm` in
tests/golden/make_golden.py).  The namespace needs RectSubdomain,
BoundaryKind, CompositeDomain, make_interface, validate and (for
non-homogeneous Dirichlet data) lift_dirichlet.

Cross geometry: five squares of N x N cells, h = 1/N: centre [0,1]^2 and
arms W/E/S/N; subdomain ids C=0, W=1, E=2, S=3, N=4 listed in that order.
Interfaces are centre <-> each arm, every other edge is ghost-node
Dirichlet whose data g = p(ghost point one spacing outside the first node
line) is lifted into the right-hand side (ref rectsolver.py:292-313).
Elongated arms (c4) keep h and use `arm` cells along the arm.
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

CENTER, WEST, EAST, SOUTH, NORTH = 0, 1, 2, 3, 4


def default_api():
    from . import geometry, rectsolver
    return SimpleNamespace(RectSubdomain=geometry.RectSubdomain,
                           BoundaryKind=geometry.BoundaryKind,
                           CompositeDomain=geometry.CompositeDomain,
                           make_interface=geometry.make_interface,
                           validate=geometry.validate,
                           lift_dirichlet=rectsolver.lift_dirichlet)


# --- manufactured solutions (numpy; evaluated on host) ---------------------

def _p_sin_exp(x, y):
    return np.sin(np.pi * x) * np.sin(np.pi * y) + np.exp(x + y) / math.e ** 2


def _lap_sin_exp(x, y):
    return -2.0 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y) \
        + 2.0 * np.exp(x + y) / math.e ** 2


def _p_sin(x, y):
    return np.sin(np.pi * x) * np.sin(np.pi * y)


def _lap_sin(x, y):
    return -2.0 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y)


SOLUTIONS = {"sin_exp": (_p_sin_exp, _lap_sin_exp), "sin": (_p_sin, _lap_sin)}


def cross_composite(N: int, arm: int | None = None, kappa: float = 0.0, api=None):
    """The BASELINE cross: centre N x N, arms N across x `arm` along, h = 1/N."""
    api = api or default_api()
    arm = N if arm is None else arm
    h = 1.0 / N
    D, I = api.BoundaryKind.DIRICHLET, api.BoundaryKind.INTERFACE

    def rect(sid, origin, m, n, iface_edge):
        bc = {e: (I if e == iface_edge or iface_edge == "all" else D)
              for e in ("west", "east", "south", "north")}
        return api.RectSubdomain(id=sid, origin=origin, m=m, n=n, dx=h, dy=h,
                                 edge_bc=bc, kappa=kappa)

    c = rect(CENTER, (0.0, 0.0), N, N, "all")
    w = rect(WEST, (-arm * h, 0.0), arm, N, "east")
    e = rect(EAST, (1.0, 0.0), arm, N, "west")
    s = rect(SOUTH, (0.0, -arm * h), N, arm, "north")
    n = rect(NORTH, (0.0, 1.0), N, arm, "south")
    ifaces = [api.make_interface(0, w, "east", c, "west"),
              api.make_interface(1, c, "east", e, "west"),
              api.make_interface(2, s, "north", c, "south"),
              api.make_interface(3, c, "north", n, "south")]
    comp = api.CompositeDomain(subdomains=[c, w, e, s, n], interfaces=ifaces)
    api.validate(comp).require()
    return comp


def node_grid(sub):
    X, Y = np.meshgrid(sub.x_nodes(), sub.y_nodes(), indexing="ij")
    return X, Y


def ghost_points(sub, edge):
    """Coordinates of the Dirichlet data one spacing outside the first line."""
    xs, ys = sub.x_nodes(), sub.y_nodes()
    if edge == "west":
        return np.full(sub.n, xs[0] - sub.dx), ys
    if edge == "east":
        return np.full(sub.n, xs[-1] + sub.dx), ys
    if edge == "south":
        return xs, np.full(sub.m, ys[0] - sub.dy)
    return xs, np.full(sub.m, ys[-1] + sub.dy)


def manufactured_rhs(comp, solution: str, api=None):
    """f = (lap p + kappa p) at nodes with every Dirichlet edge lifted."""
    api = api or default_api()
    p, lap = SOLUTIONS[solution]
    D = api.BoundaryKind.DIRICHLET
    f, exact = {}, {}
    for sub in comp.subdomains:
        X, Y = node_grid(sub)
        rhs = (lap(X, Y) + sub.kappa * p(X, Y)).ravel()
        for edge in ("west", "east", "south", "north"):
            if sub.edge_bc[edge] is D:
                gx, gy = ghost_points(sub, edge)
                rhs = api.lift_dirichlet(sub, rhs, edge, p(gx, gy))
        f[sub.id] = np.ascontiguousarray(rhs)
        exact[sub.id] = p(X, Y).ravel()
    return f, exact


_SOLUTION_CODE = {"sin_exp": 0, "sin": 1}


def manufactured_rhs_device(comp, solution: str):
    """manufactured_rhs assembled on the device (C ABI fd_assemble_rhs, SURVEY
    8f row 3): the same recipe -- f = lap p + kappa p at the nodes, each
    Dirichlet edge lifted with p at its ghost points -- without the host
    arrays or their upload.  Returns ({id: f}, {id: exact}) as CUDA tensors."""
    import torch

    from . import _native
    from .geometry import BoundaryKind
    _native.require_cuda()
    f, exact = {}, {}
    for sub in comp.subdomains:
        lift = []
        for edge in ("west", "east", "south", "north"):
            if sub.edge_bc[edge] is BoundaryKind.DIRICHLET:
                lift.append(2.0 if edge in sub.half_cell_dirichlet else 1.0)
            else:
                lift.append(0.0)
        fi = torch.empty(sub.size, dtype=torch.float64, device="cuda")
        ei = torch.empty(sub.size, dtype=torch.float64, device="cuda")
        _native.call("fd_assemble_rhs", sub.m, sub.n, float(sub.origin[0]), float(sub.origin[1]),
                     float(sub.dx), float(sub.dy), float(sub.kappa), _SOLUTION_CODE[solution], *lift,
                     _native.dptr(fi), _native.dptr(ei), _native.stream_ptr())
        f[sub.id], exact[sub.id] = fi, ei
    return f, exact


def rel_l2_device(fields: dict, exact: dict) -> float:
    """rel_l2 with both sides on the device."""
    num = den = 0.0
    for sid, ex in exact.items():
        v = fields[sid]
        v = v.values if hasattr(v, "values") else v
        num += float(((v - ex) ** 2).sum())
        den += float((ex ** 2).sum())
    return math.sqrt(num / den)


def random_rhs(comp, seed: int = 0):
    """i.i.d. uniform[-1, 1] per subdomain, drawn in id order from one generator."""
    rng = np.random.default_rng(seed)
    return {sub.id: rng.uniform(-1.0, 1.0, sub.size)
            for sub in sorted(comp.subdomains, key=lambda s: s.id)}


def build_cross_case(name: str, api=None, N: int | None = None, device: bool = False):
    """(composite, rhs dict, exact dict or None, meta) for c0, c2, c3, c4 or a
    reduced-N variant of their geometry (`N` overrides the size).  device=True
    assembles the manufactured right-hand sides (c0, c2, c4) on the GPU."""
    api = api or default_api()
    if name in ("c0", "c2"):
        N = N or (141 if name == "c0" else 2047)
        comp = cross_composite(N, kappa=0.0, api=api)
        f, exact = manufactured_rhs_device(comp, "sin_exp") if device else manufactured_rhs(comp, "sin_exp", api)
    elif name == "c3":
        N = N or 4095
        comp = cross_composite(N, kappa=-100.0, api=api)
        f, exact = random_rhs(comp, 0), None
    elif name == "c4":
        N = N or 4095
        arm = 4 * N + 3          # 16383 at N = 4095: same h, n stays 2^p - 1
        comp = cross_composite(N, arm=arm, kappa=0.0, api=api)
        f, exact = manufactured_rhs_device(comp, "sin") if device else manufactured_rhs(comp, "sin", api)
    else:
        raise ValueError(f"unknown cross config {name!r}")
    meta = {"name": name, "N": N, "points": sum(s.size for s in comp.subdomains),
            "gmres_m": 50, "tol": 1e-10}
    return comp, f, exact, meta


def reference_cross(k_n: int, L: float = 1.0 / 7.0, kappa: float = 0.0, api=None):
    """The reference package's own five-rectangle test cross (its bench.py
    build_cross: side L, k_n nodes per L, h = L/k_n), restated on the geometry
    API: a 2L x 4L centre with interfaces on all sides; west/east arms with
    Neumann flanks (south/north) and a half-cell Dirichlet far end; south/north
    arms with Neumann flanks (west/east) and a half-cell Dirichlet far end.  The
    arms' transform axes are NN pairs (y for west/east, x for south/north)."""
    api = api or default_api()
    D, N, I = api.BoundaryKind.DIRICHLET, api.BoundaryKind.NEUMANN, api.BoundaryKind.INTERFACE
    h, k = L / k_n, k_n

    def rect(sid, origin, m, n, bc, half=()):
        return api.RectSubdomain(id=sid, origin=origin, m=m, n=n, dx=h, dy=h, edge_bc=bc, kappa=kappa,
                                 half_cell_dirichlet=frozenset(half))

    c = rect(CENTER, (L, 2 * L), 2 * k, 4 * k, {"west": I, "east": I, "south": I, "north": I})
    w = rect(WEST, (0.0, 2 * L), k, 4 * k, {"west": D, "east": I, "south": N, "north": N}, ("west",))
    e = rect(EAST, (3 * L, 2 * L), 4 * k, 4 * k, {"west": I, "east": D, "south": N, "north": N}, ("east",))
    s_ = rect(SOUTH, (L, 0.0), 2 * k, 2 * k, {"west": N, "east": N, "south": D, "north": I}, ("south",))
    n_ = rect(NORTH, (L, 6 * L), 2 * k, k, {"west": N, "east": N, "south": I, "north": D}, ("north",))
    ifaces = [api.make_interface(0, w, "east", c, "west"), api.make_interface(1, c, "east", e, "west"),
              api.make_interface(2, s_, "north", c, "south"), api.make_interface(3, c, "north", n_, "south")]
    comp = api.CompositeDomain(subdomains=[c, w, e, s_, n_], interfaces=ifaces)
    api.validate(comp).require()
    return comp


def _psi_coeffs(L: float):
    """Phase polynomials of the reference cross's manufactured solution
    (reference bench.py derive_psi_coeffs): psi_x(x) = x (A1 + A2 (x - L) +
    A3 (x^2 - 4 L x + 3 L^2)) hits pi/2, 3pi/2, 3pi at x = L, 3L, 7L and psi_y
    hits pi/2, 3pi/2, 2pi at y = 2L, 6L, 7L (3 x 3 solves per axis), so
    p = sin psi_x sin psi_y vanishes on the outer Dirichlet edges."""
    def axis(xs, targets, shift, q):
        M = np.array([[x, x * (x - shift), x * q(x)] for x in xs])
        return np.linalg.solve(M, np.asarray(targets))
    a = axis([L, 3 * L, 7 * L], [np.pi / 2, 3 * np.pi / 2, 3 * np.pi], L, lambda x: x * x - 4 * L * x + 3 * L * L)
    b = axis([2 * L, 6 * L, 7 * L], [np.pi / 2, 3 * np.pi / 2, 2 * np.pi], 2 * L,
             lambda y: y * y - 8 * L * y + 12 * L * L)
    return a, b


def reference_cross_case(k_n: int, L: float = 1.0 / 7.0, kappa: float = 0.0, api=None):
    """reference_cross(k_n) with its manufactured problem (reference bench.py
    manufactured_solution / manufactured_rhs / rhs_fields): f = Laplacian of
    p = sin psi_x(x) sin psi_y(y) (+ kappa p) at the nodes, no lifting (p is
    zero on the Dirichlet edges).  Returns (comp, f, exact)."""
    comp = reference_cross(k_n, L, kappa, api)
    (A1, A2, A3), (B1, B2, B3) = _psi_coeffs(L)
    f, exact = {}, {}
    for sub in comp.subdomains:
        x, y = (a.ravel() for a in node_grid(sub))
        px = x * (A1 + A2 * (x - L) + A3 * (x * x - 4 * L * x + 3 * L * L))
        dpx = A1 + A2 * (2 * x - L) + A3 * (3 * x * x - 8 * L * x + 3 * L * L)
        ddpx = 2 * A2 + A3 * (6 * x - 8 * L)
        py = y * (B1 + B2 * (y - 2 * L) + B3 * (y * y - 8 * L * y + 12 * L * L))
        dpy = B1 + B2 * (2 * y - 2 * L) + B3 * (3 * y * y - 16 * L * y + 12 * L * L)
        ddpy = 2 * B2 + B3 * (6 * y - 16 * L)
        sx, cx, sy, cy = np.sin(px), np.cos(px), np.sin(py), np.cos(py)
        rhs = (ddpx * cx - dpx * dpx * sx) * sy + sx * (ddpy * cy - dpy * dpy * sy)
        if kappa:
            rhs = rhs + kappa * sx * sy
        f[sub.id] = rhs
        exact[sub.id] = sx * sy
    return comp, f, exact


def batch_rects(n: int = 1023, count: int = 5, kappa: float = 0.0, api=None):
    """c1: `count` independent all-Dirichlet n x n rectangles, h = 1/n."""
    api = api or default_api()
    D = api.BoundaryKind.DIRICHLET
    bc = {e: D for e in ("west", "east", "south", "north")}
    return [api.RectSubdomain(id=i, origin=(0.0, 0.0), m=n, n=n, dx=1.0 / n,
                              dy=1.0 / n, edge_bc=bc, kappa=kappa) for i in range(count)]


def rel_l2(fields: dict, exact: dict) -> float:
    """||num - exact||_2 / ||exact||_2 over all nodes of all subdomains."""
    num = den = 0.0
    for sid, ex in exact.items():
        v = fields[sid]
        v = v.values if hasattr(v, "values") else v
        v = v.detach().cpu().numpy() if hasattr(v, "detach") else np.asarray(v)
        d = v - ex
        num += float(d @ d)
        den += float(ex @ ex)
    return math.sqrt(num / den)
