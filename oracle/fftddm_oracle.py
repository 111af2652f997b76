"""CPU ORACLE — TEST INFRASTRUCTURE ONLY, NEVER A PRODUCT PATH.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module.  The package
`paper_2509_23180_b200` never imports it and has no CPU fallback.

What it is: a numpy restatement of the reference `fftddm` hot path for the
configurations the GPU path supports (DD or NN transform axis, along y or --
with the field transposed -- along x, any per-end diagonal modification on
the sweep axis), written from the reference's algorithm description.  Each function cites the reference
file:line it follows (paths relative to /root/reference/pkg/src/fftddm/).
It uses the same numpy primitives as the reference (numpy's pocketfft for
the DST-I, numpy BLAS for dots), so its timing stands in for the reference
solver on the GPU box, where /root/reference does not exist.

Pinning: tests/test_oracle_golden.py checks every function here against
fixtures written by the real reference (tests/golden/make_golden.py
imports /root/reference in the build container) and against the
reference's own known-answer tests.  Parity status:
PINNED.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

PIVOT_RTOL = 1e-13          # rectsolver.py:21
BREAKDOWN = 1e-14           # krylov.py:27


# --- transforms --------------------------------------------------------------

def eigenvalues_dd(n, delta_t, delta_o, kappa=0.0):
    """lambda_j = -2(dt+do) + 2 dt cos(j pi/(n+1)) + kappa   (transforms.py:26-31,38)."""
    j = np.arange(1, n + 1, dtype=float)
    return -2.0 * (delta_t + delta_o) + 2.0 * delta_t * np.cos(j * np.pi / (n + 1)) + kappa


def eigenvalues(bc, n, delta_t, delta_o, kappa=0.0):
    """DD: cos(j pi/(n+1)); NN: cos((j-1) pi/n); PP: cos(2 pi (j-1)/n)
    (transforms.py:26-38)."""
    if bc == "DD":
        return eigenvalues_dd(n, delta_t, delta_o, kappa)
    j = np.arange(1, n + 1, dtype=float)
    if bc == "NN":
        c = np.cos((j - 1) * np.pi / n)
    elif bc == "PP":
        c = np.cos(2.0 * np.pi * (j - 1) / n)
    else:
        raise NotImplementedError(f"unknown pair {bc}")
    return -2.0 * (delta_t + delta_o) + 2.0 * delta_t * c + kappa


def dct2(v):
    """sum_k v_k cos(pi j (2k+1)/(2n)) through the even extension of length 2n
    and one complex FFT, phase-shifted                  (transforms.py:83-89)."""
    n = v.shape[-1]
    ext = np.concatenate([v, v[..., ::-1]], axis=-1)
    spec = np.fft.fft(ext, axis=-1)[..., :n]
    return 0.5 * (np.exp(-0.5j * np.pi * np.arange(n) / n) * spec).real


def dct3(a):
    """sum_j a_j cos(pi j (2k+1)/(2n)) through one length-2n inverse FFT
    (transforms.py:92-97)."""
    n = a.shape[-1]
    z = np.zeros(a.shape[:-1] + (2 * n,), dtype=complex)
    z[..., :n] = a * np.exp(0.5j * np.pi * np.arange(n) / n)
    return 2 * n * np.fft.ifft(z, axis=-1).real[..., :n]


def nn_scale(n):
    """sqrt(1/n) for the constant mode, sqrt(2/n) otherwise   (transforms.py:100-103)."""
    s = np.full(n, math.sqrt(2.0 / n))
    s[0] = math.sqrt(1.0 / n)
    return s


def apply_q_pp(v):
    """Real Fourier basis: cosine amplitudes to the real part, sine amplitudes
    to the imaginary part of a half spectrum, one inverse FFT (transforms.py:114-126)."""
    n = v.shape[-1]
    spec = np.zeros(v.shape[:-1] + (n,), dtype=complex)
    root = math.sqrt(1.0 / n)
    spec[..., 0] = v[..., 0] * root
    spec[..., n // 2] = v[..., n // 2] * root
    if n > 2:
        amp = math.sqrt(2.0 / n)
        spec[..., 1:n // 2] = amp * v[..., 1:n // 2]
        spec[..., n // 2 + 1:] = -1j * amp * v[..., n // 2 + 1:]
    return n * np.fft.ifft(spec, axis=-1).real


def apply_qt_pp(v):
    """Q^T of the real Fourier basis through one FFT (transforms.py:139-148)."""
    n = v.shape[-1]
    spec = np.fft.fft(v, axis=-1)
    out = np.empty_like(v)
    root = math.sqrt(1.0 / n)
    out[..., 0] = spec[..., 0].real * root
    out[..., n // 2] = spec[..., n // 2].real * root
    if n > 2:
        amp = math.sqrt(2.0 / n)
        out[..., 1:n // 2] = amp * spec[..., 1:n // 2].real
        out[..., n // 2 + 1:] = -amp * spec[..., n // 2 + 1:].imag
    return out


def apply_q(bc, v):
    """Q v along the last axis (transforms.py:106-126)."""
    v = np.asarray(v, dtype=float)
    if bc == "PP":
        return apply_q_pp(v)
    return apply_q_dd(v) if bc == "DD" else dct3(nn_scale(v.shape[-1]) * v)


def apply_qt(bc, v):
    """Q^T v along the last axis (transforms.py:129-148)."""
    v = np.asarray(v, dtype=float)
    if bc == "PP":
        return apply_qt_pp(v)
    return apply_q_dd(v) if bc == "DD" else nn_scale(v.shape[-1]) * dct2(v)


def dst1(v):
    """sum_k v_k sin(j k pi/(n+1)) along the last axis through the odd
    extension of length 2(n+1) and one complex FFT       (transforms.py:74-80)."""
    n = v.shape[-1]
    ext = np.zeros(v.shape[:-1] + (2 * n + 2,))
    ext[..., 1:n + 1] = v
    ext[..., n + 2:] = -v[..., ::-1]
    spec = np.fft.fft(ext, axis=-1)
    return -0.5 * spec.imag[..., 1:n + 1]


def apply_q_dd(v):
    """Orthonormal DD eigenbasis, Q = Q^T = sqrt(2/(n+1)) DST-I
    (transforms.py:112-113,135-136)."""
    n = v.shape[-1]
    return math.sqrt(2.0 / (n + 1)) * dst1(np.asarray(v, dtype=float))


# --- rectangle solver ---------------------------------------------------------

def factor_tridiag(diag, off, tol):
    """Per-column LU of tridiag(off, diag, off) with the reference's pivot
    guard: returns (beta, lower, bad)                   (rectsolver.py:62-77)."""
    ms = diag.shape[0]
    beta = np.empty_like(diag)
    lower = np.zeros_like(diag)
    beta[0] = diag[0]
    bad = np.abs(beta[0]) < tol
    piv = np.where(bad, 1.0, beta[0])
    for i in range(1, ms):
        lower[i] = off / piv
        beta[i] = diag[i] - off * lower[i]
        bad = bad | (np.abs(beta[i]) < tol)
        piv = np.where(bad, 1.0, beta[i])
        beta[i] = piv
    return beta, lower, bad


def tridiag_solve(beta, lower, off, rhs):
    """Forward y_i = r_i - l_i y_{i-1}; back x_i = (y_i - off x_{i+1})/beta_i
    (rectsolver.py:80-91)."""
    ms = rhs.shape[0]
    y = np.empty_like(rhs)
    y[0] = rhs[0]
    for i in range(1, ms):
        y[i] = rhs[i] - lower[i] * y[i - 1]
    x = np.empty_like(rhs)
    x[ms - 1] = y[ms - 1] / beta[ms - 1]
    for i in range(ms - 2, -1, -1):
        x[i] = (y[i] - off * x[i + 1]) / beta[i]
    return x


class SingularOracleError(Exception):
    pass


@dataclass
class OraclePlan:
    sub: object
    beta: np.ndarray
    lower: np.ndarray
    off: float
    axis: str = "y"
    bc: str = "DD"
    cyclic: bool = False
    sm_q: np.ndarray = None
    sm_denom: np.ndarray = None
    sm_gamma: np.ndarray = None
    singular: tuple = ()
    singular_dense: tuple = ()


def transformable(sub, axis):
    """Pure form: NN or PP, or DD with ghost-node ends   (rectsolver.py:24-29)."""
    pair = sub.axis_pair(axis)
    if pair in ("NN", "PP"):
        return True
    lo, hi = ("west", "east") if axis == "x" else ("south", "north")
    return pair == "DD" and sub.end_modifier(lo) == 0.0 and sub.end_modifier(hi) == 0.0


def plan(sub, axis=None, pin_mean=False):
    """plan_rect (rectsolver.py:94-180): axis y when transformable, else x (the
    field is transposed, rectsolver.py:198-199); `axis` forces the choice.  A
    periodic sweep axis factors the rank-one modified system and keeps the
    Sherman-Morrison correction solves (rectsolver.py:136-153); pin_mean keeps
    the dense matrices of singular modes (rectsolver.py:157-175)."""
    if axis is None:
        axis = "y" if transformable(sub, "y") else "x"
    if not transformable(sub, axis):
        raise NotImplementedError(f"axis {axis} is not transformable")
    if axis == "y":
        nt, ms, dt, ds, lo, hi = sub.n, sub.m, sub.delta_y, sub.delta_x, "west", "east"
    else:
        nt, ms, dt, ds, lo, hi = sub.m, sub.n, sub.delta_x, sub.delta_y, "south", "north"
    bc = sub.axis_pair(axis)
    cyclic = sub.axis_pair("x" if axis == "y" else "y") == "PP"
    lam = eigenvalues(bc, nt, dt, ds, sub.kappa)
    diag = np.tile(lam, (ms, 1))
    if cyclic:
        if ms % 2:
            raise SingularOracleError("periodic sweep axis needs an even count")
    else:
        diag[0] += sub.end_modifier(lo)
        diag[-1] += sub.end_modifier(hi)
    tol = PIVOT_RTOL * max(np.abs(lam).max(), ds)
    q = den = gam = None
    if cyclic and ms > 2:
        gam = np.where(np.abs(diag[0]) > tol, -diag[0], ds)
        bd = diag.copy()
        bd[0] -= gam
        bd[-1] -= ds * ds / gam
        beta, lower, bad = factor_tridiag(bd, ds, tol)
        u = np.zeros((ms, nt))
        u[0] = gam
        u[-1] = ds
        q = tridiag_solve(beta, lower, ds, u)
        den = 1.0 + q[0] + (ds / gam) * q[-1]
        bad = bad | (np.abs(den) < 1e-12)
    elif cyclic:
        beta, lower, bad = factor_tridiag(diag, 2.0 * ds, tol)
    else:
        beta, lower, bad = factor_tridiag(diag, ds, tol)
    singular, mats = (), ()
    if np.any(bad):
        if not pin_mean:
            raise SingularOracleError(f"singular modes {np.nonzero(bad)[0].tolist()}")
        singular = tuple(int(k) for k in np.nonzero(bad)[0])
        ms_list = []
        for k in singular:
            M = np.diag(diag[:, k])
            i = np.arange(ms - 1)
            M[i, i + 1] += ds
            M[i + 1, i] += ds
            if cyclic:
                M[0, ms - 1] += ds
                M[ms - 1, 0] += ds
            ms_list.append(M)
        mats = tuple(ms_list)
    return OraclePlan(sub=sub, beta=beta, lower=lower, off=ds, axis=axis, bc=bc, cyclic=cyclic,
                      sm_q=q, sm_denom=den, sm_gamma=gam, singular=singular, singular_dense=mats)


def solve(pl: OraclePlan, f):
    """Q^T along the transform axis -> per-mode tridiagonal (+ periodic
    correction, + minimum-norm singular modes) -> Q   (rectsolver.py:183-213)."""
    grid = np.asarray(f, dtype=float).reshape(pl.sub.m, pl.sub.n)
    if pl.axis == "x":
        grid = grid.T
    fhat = apply_qt(pl.bc, grid)
    off = 2.0 * pl.off if (pl.cyclic and fhat.shape[0] == 2) else pl.off
    phat = tridiag_solve(pl.beta, pl.lower, off, fhat)
    if pl.sm_q is not None:
        vy = phat[0] + (pl.off / pl.sm_gamma) * phat[-1]
        phat = phat - pl.sm_q * (vy / pl.sm_denom)
    for k, M in zip(pl.singular, pl.singular_dense):
        phat[:, k] = np.linalg.lstsq(M, fhat[:, k], rcond=None)[0]
    out = apply_q(pl.bc, phat)
    if pl.axis == "x":
        out = out.T
    return np.ascontiguousarray(out).reshape(-1)


def apply_operator(sub, v):
    """5-point matvec with end modifiers or periodic wrap (rectsolver.py:264-289)."""
    G = np.asarray(v, dtype=float).reshape(sub.m, sub.n)
    dx, dy = sub.delta_x, sub.delta_y
    out = (-2.0 * (dx + dy) + sub.kappa) * G
    out[:, 1:] += dy * G[:, :-1]
    out[:, :-1] += dy * G[:, 1:]
    if sub.axis_pair("y") == "PP":
        out[:, 0] += dy * G[:, -1]
        out[:, -1] += dy * G[:, 0]
    else:
        out[:, 0] += sub.end_modifier("south") * G[:, 0]
        out[:, -1] += sub.end_modifier("north") * G[:, -1]
    out[1:, :] += dx * G[:-1, :]
    out[:-1, :] += dx * G[1:, :]
    if sub.axis_pair("x") == "PP":
        out[0, :] += dx * G[-1, :]
        out[-1, :] += dx * G[0, :]
    else:
        out[0, :] += sub.end_modifier("west") * G[0, :]
        out[-1, :] += sub.end_modifier("east") * G[-1, :]
    return out.reshape(-1)


# --- Schur operator -----------------------------------------------------------

def _line(sub, edge):
    m, n = sub.m, sub.n
    return {"west": np.arange(n), "east": (m - 1) * n + np.arange(n),
            "south": np.arange(m) * n, "north": np.arange(m) * n + (n - 1)}[edge]


@dataclass
class Coupling:
    """R: `to[to_idx] = coupling * from[from_idx]`    (ddm.py:27-70)."""
    from_idx: np.ndarray
    to_idx: np.ndarray
    to_size: int
    coupling: float

    def apply(self, v):
        out = np.zeros(self.to_size)
        out[self.to_idx] = self.coupling * v[self.from_idx]
        return out


def coupling(comp, iface, from_id):
    to_id = iface.other_side(from_id)[0]
    sf, st = comp.subdomain(from_id), comp.subdomain(to_id)
    perm = np.asarray(iface.index_map)
    if iface.side_a[0] == from_id:
        fi, ti = _line(sf, iface.side_a[1]), _line(st, iface.side_b[1])[perm]
    else:
        fi, ti = _line(sf, iface.side_b[1])[perm], _line(st, iface.side_a[1])
    return Coupling(fi, ti, st.size, iface.coupling)


class Schur:
    """Matrix-free (A_c - sum_i R_ci A_i^-1 R_ic) on the centre (ddm.py:94-136)."""

    def __init__(self, comp, coupled_id=None, threads=1):
        # threads > 1: neighbour solves on a pool, like the reference's
        # ThreadPoolExecutor over arms (ddm.py:182-201, 112-123)
        self.pool = None
        if coupled_id is None:
            ids = sorted(comp.coupled_ids)
            coupled_id = ids[0] if ids else min(s.id for s in comp.subdomains)
        self.coupled_id = coupled_id
        self.center = comp.subdomain(coupled_id)
        self.center_plan = plan(self.center)
        self.neighbors = []
        for f in comp.interfaces_of(coupled_id):
            other = f.other_side(coupled_id)[0]
            self.neighbors.append((plan(comp.subdomain(other)),
                                   coupling(comp, f, other),          # R_ci
                                   coupling(comp, f, coupled_id)))    # R_ic
        if threads > 1 and len(self.neighbors) > 1:
            from concurrent.futures import ThreadPoolExecutor
            self.pool = ThreadPoolExecutor(max_workers=min(threads, len(self.neighbors)))

    @property
    def size(self):
        return self.center.size

    def schur(self, p):
        out = np.zeros(self.size)
        if self.pool is not None:   # solves in parallel, parts added in neighbour order
            parts = list(self.pool.map(lambda nb: nb[1].apply(solve(nb[0], nb[2].apply(p))), self.neighbors))
            for part in parts:
                out += part
            return out
        for pl, to_c, from_c in self.neighbors:
            out += to_c.apply(solve(pl, from_c.apply(p)))
        return out

    def center_solve(self, r):
        return solve(self.center_plan, r)

    def preconditioned(self, p):
        return p - self.center_solve(self.schur(p))

    def unpreconditioned(self, p):
        return apply_operator(self.center, p) - self.schur(p)


# --- GMRES ---------------------------------------------------------------------

@dataclass
class Report:
    converged: bool
    iterations: int
    residual_history: np.ndarray
    wall_time: float
    true_residual: float = float("nan")


def gmres(op, rhs, m=80, tol=1e-10, max_restarts=200, x0=None):
    """Restarted GMRES(m), MGS Arnoldi, Givens LSQ (krylov.py:61-165).
    Returns (x, Report); raises RuntimeError on non-convergence."""
    t0 = time.perf_counter()
    N = rhs.size
    x = np.zeros(N) if x0 is None else np.array(x0, dtype=float)
    r = rhs - op(x) if x.any() else rhs.copy()
    r0 = np.linalg.norm(r)
    if r0 == 0.0:
        return x, Report(True, 0, np.zeros(1), time.perf_counter() - t0)
    hist = [1.0]
    its = 0
    m = min(m, N)
    for _ in range(max_restarts):
        beta = np.linalg.norm(r)
        if beta / r0 <= tol:
            break
        V = np.empty((m + 1, N))
        H = np.zeros((m + 1, m))
        V[0] = r / beta
        g = np.zeros(m + 1)
        g[0] = beta
        cs, sn = np.zeros(m), np.zeros(m)
        used, broke = 0, False
        for k in range(m):
            w = np.array(op(V[k]), dtype=float)
            wn = np.linalg.norm(w)
            for i in range(k + 1):
                H[i, k] = V[i] @ w
                w -= H[i, k] * V[i]
            hn = np.linalg.norm(w)
            H[k + 1, k] = hn
            for i in range(k):
                a, b = H[i, k], H[i + 1, k]
                H[i, k] = cs[i] * a + sn[i] * b
                H[i + 1, k] = -sn[i] * a + cs[i] * b
            rho = np.hypot(H[k, k], H[k + 1, k])
            cs[k] = H[k, k] / rho if rho else 1.0
            sn[k] = H[k + 1, k] / rho if rho else 0.0
            H[k, k], H[k + 1, k] = rho, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            its += 1
            used = k + 1
            hist.append(abs(g[k + 1]) / r0)
            if hn <= BREAKDOWN * wn or hn == 0.0:
                broke = True
                break
            V[k + 1] = w / hn
            if hist[-1] <= tol:
                break
        y = np.zeros(used)
        for i in range(used - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:used] @ y[i + 1:used]) / H[i, i]
        x = x + V[:used].T @ y
        r = rhs - op(x)
        rel = np.linalg.norm(r) / r0
        if rel <= tol or (broke and hist[-1] <= tol):
            hist[-1] = rel
            return x, Report(True, its, np.asarray(hist), time.perf_counter() - t0,
                             float(np.linalg.norm(r)))
        if broke:
            break
    raise RuntimeError(f"oracle GMRES did not converge in {its} iterations")


def ddm_solve(comp, f, m=50, tol=1e-10, max_restarts=200, threads=1):
    """Algorithm 1: arm pre-solves, reduced RHS, GMRES on the preconditioned
    Schur system, back-substitution (ddm.py:210-270, krylov.py:168-195)."""
    op = Schur(comp, threads=threads)
    qs = [solve(pl, np.asarray(f[pl.sub.id], dtype=float)) for pl, _, _ in op.neighbors]
    fp = np.array(f[op.coupled_id], dtype=float)
    for (pl, to_c, _), q in zip(op.neighbors, qs):
        fp -= to_c.apply(q)
    x, rep = gmres(op.preconditioned, op.center_solve(fp), m=m, tol=tol,
                   max_restarts=max_restarts)
    rep.true_residual = float(np.linalg.norm(op.unpreconditioned(x) - fp))
    out = {op.coupled_id: x}
    for (pl, _, from_c), q in zip(op.neighbors, qs):
        out[pl.sub.id] = q - solve(pl, from_c.apply(x))
    return out, rep
