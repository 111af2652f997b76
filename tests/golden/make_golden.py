"""Generate the parity fixtures in tests/golden/ by running the REAL reference.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py small c0 c1 nn cyclic   # seconds
    python tests/golden/make_golden.py c2 c3              # minutes (c3 ~15 min, 16 GB)

The reference package is imported from /root/reference/pkg/src; its inputs
come from paper_2509_23180_b200.configs driven with the *reference's*
geometry API (api=fftddm), so the GPU tests rebuild bit-identical inputs from
the same recipe.  Large fields are stored as norms plus values at fixed
sampled indices; c0 and the small cases are stored in full.
"""

from __future__ import annotations

import os
import sys
import time
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import fftddm                                          # noqa: E402  (the reference)
from fftddm import ddm, geometry, krylov, rectsolver, transforms  # noqa: E402
from paper_2509_23180_b200 import configs              # noqa: E402

API = SimpleNamespace(RectSubdomain=geometry.RectSubdomain, BoundaryKind=geometry.BoundaryKind,
                      CompositeDomain=geometry.CompositeDomain,
                      make_interface=geometry.make_interface, validate=geometry.validate,
                      lift_dirichlet=rectsolver.lift_dirichlet)
B = geometry.BoundaryKind
SAMPLES = 4096


def sample_idx(size, sid):
    rng = np.random.default_rng(1000 + sid)
    k = min(SAMPLES, size)
    return np.sort(rng.choice(size, k, replace=False))


def rect(m, n, dx, dy, kappa, bc, half=()):
    kinds = {"D": B.DIRICHLET, "N": B.NEUMANN, "I": B.INTERFACE, "P": B.PERIODIC}
    edge_bc = {e: kinds[c] for e, c in zip(("west", "east", "south", "north"), bc)}
    return geometry.RectSubdomain(id=0, origin=(0.0, 0.0), m=m, n=n, dx=dx, dy=dy,
                                  edge_bc=edge_bc, kappa=kappa,
                                  half_cell_dirichlet=frozenset(half))


# (m, n, dx, dy, kappa, bc WESN, half-cell edges) -- all DD along y
RECT_CASES = [
    (1, 1, 1.0, 1.0, 0.0, "DDDD", ()),
    (3, 3, 1.0, 1.0, 0.0, "DDDD", ()),
    (5, 4, 0.5, 0.25, -1.5, "DDDD", ()),
    (8, 7, 1.0 / 8, 1.0 / 8, 0.0, "DDDD", ()),
    (16, 15, 1.0 / 16, 1.0 / 16, -10.0, "DDDD", ()),
    (33, 31, 1.0 / 31, 1.0 / 31, 0.0, "DDDD", ()),
    (64, 63, 1.0 / 64, 1.0 / 64, 3.0, "DDDD", ()),
    (20, 127, 0.01, 0.02, -100.0, "DDDD", ()),
    (141, 141, 1.0 / 141, 1.0 / 141, 0.0, "DDDD", ()),
    (12, 9, 1.0, 1.0, 0.0, "DDDD", ("west",)),
    (12, 9, 1.0, 1.0, 0.0, "DDDD", ("west", "east")),
    (10, 15, 0.1, 0.1, -2.0, "NNDD", ()),
    (9, 31, 1.0, 0.5, 0.0, "IDDD", ("east",)),
    (257, 255, 1.0 / 255, 1.0 / 255, 0.0, "DDDD", ()),
    (40, 1023, 1.0 / 1023, 1.0 / 1023, -10.0, "DDDD", ()),
]


def make_small():
    out = {}
    rng = np.random.default_rng(7)
    # DST-I / apply_Q on row batches (transforms.py:106-113)
    for n in (1, 2, 3, 4, 7, 8, 15, 31, 63, 64, 127, 141, 255, 511, 1023, 2047, 4095):
        x = rng.standard_normal((3, n))
        pl = transforms.make_plan("DD", n, 1.0, 1.0)
        out[f"dst_in_{n}"] = x
        out[f"dst_out_{n}"] = transforms.apply_Q(pl, x)
        out[f"eig_{n}"] = transforms.eigenvalues("DD", n, 2.5, 0.75, kappa=-0.5)
    # rectangle plans and solves (rectsolver.py:94-213,264-289)
    for c, (m, n, dx, dy, kappa, bc, half) in enumerate(RECT_CASES):
        sub = rect(m, n, dx, dy, kappa, bc, half)
        pl = rectsolver.plan_rect(sub)
        f = rng.uniform(-1, 1, m * n)
        out[f"rect_f_{c}"] = f
        out[f"rect_p_{c}"] = rectsolver.solve_rect(pl, f).values
        if m * n <= 5000:
            out[f"rect_beta_{c}"] = pl.beta
            out[f"rect_lower_{c}"] = pl.lower
        out[f"rect_Av_{c}"] = rectsolver.apply_rect_operator(sub, f)
    # BASELINE-geometry crosses at reduced N: Schur applies + full solves
    for N in (4, 8, 15, 31):
        for kappa in (0.0, -100.0):
            tag = f"{N}_{int(-kappa)}"
            comp = configs.cross_composite(N, kappa=kappa, api=API)
            op = ddm.build_schur_operator(comp, threads=1)
            p = rng.standard_normal(op.size)
            out[f"x_p_{tag}"] = p
            out[f"x_schur_{tag}"] = op.schur(p)
            out[f"x_pre_{tag}"] = op.preconditioned(p)
            out[f"x_unpre_{tag}"] = op.unpreconditioned(p)
            f, exact = configs.manufactured_rhs(comp, "sin_exp", api=API)
            fields, rep = ddm.ddm_solve(comp, f, krylov.GmresConfig(m=50, tol=1e-10))
            for sid, fld in fields.items():
                out[f"x_sol_{tag}_{sid}"] = fld.values
            out[f"x_iters_{tag}"] = np.array(rep.iterations)
            out[f"x_hist_{tag}"] = rep.residual_history
            out[f"x_true_{tag}"] = np.array(rep.true_residual)
    # GMRES on a dense well-conditioned system with a small restart (krylov.py:61-165)
    A = np.eye(40) + 0.3 * rng.standard_normal((40, 40)) / np.sqrt(40)
    b = rng.standard_normal(40)
    x, rep = krylov.gmres(lambda v: A @ v, b, cfg=krylov.GmresConfig(m=7, tol=1e-12))
    out.update(gm_A=A, gm_b=b, gm_x=x, gm_iters=np.array(rep.iterations),
               gm_hist=rep.residual_history)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small.npz", len(out), "arrays")


def solve_cross(name, full):
    t0 = time.perf_counter()
    comp, f, exact, meta = configs.build_cross_case(name, api=API)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    fields, rep = ddm.ddm_solve(comp, f, krylov.GmresConfig(m=50, tol=1e-10))
    wall = time.perf_counter() - t0
    out = dict(iterations=np.array(rep.iterations), history=rep.residual_history,
               true_residual=np.array(rep.true_residual), wall=np.array(wall),
               build=np.array(t_build), threads=np.array(ddm.solver_threads()),
               points=np.array(meta["points"]))
    if exact is not None:
        out["rel_l2_exact"] = np.array(configs.rel_l2(fields, exact))
    for sid, fld in fields.items():
        v = fld.values
        out[f"norm_{sid}"] = np.array(np.linalg.norm(v))
        out[f"sum_{sid}"] = np.array(v.sum())
        idx = sample_idx(v.size, sid)
        out[f"idx_{sid}"] = idx
        out[f"val_{sid}"] = v[idx]
        if full:
            out[f"sol_{sid}"] = v
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "iters", rep.iterations, "wall", round(wall, 2), "s",
          "rel_l2", out.get("rel_l2_exact"))


def make_c1():
    out = {}
    for kappa in (0.0, -10.0):
        subs = configs.batch_rects(1023, 5, kappa, api=API)
        rng = np.random.default_rng(0)
        f = [rng.uniform(-1, 1, s.size) for s in subs]
        plans = [rectsolver.plan_rect(s) for s in subs]
        t0 = time.perf_counter()
        ps = [rectsolver.solve_rect(pl, fi).values for pl, fi in zip(plans, f)]
        out[f"wall_{int(-kappa)}"] = np.array(time.perf_counter() - t0)
        for sid, v in enumerate(ps):
            idx = sample_idx(v.size, sid)
            out[f"idx_{int(-kappa)}_{sid}"] = idx
            out[f"val_{int(-kappa)}_{sid}"] = v[idx]
            out[f"norm_{int(-kappa)}_{sid}"] = np.array(np.linalg.norm(v))
            out[f"sum_{int(-kappa)}_{sid}"] = np.array(v.sum())
            out[f"row0_{int(-kappa)}_{sid}"] = v[:1023]
            out[f"rowlast_{int(-kappa)}_{sid}"] = v[-1023:]
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)
    print("c1.npz written")


# NN-transform rectangles (m, n, dx, dy, kappa, bc WESN, half-cell edges): the
# reference picks y when y is NN or ghost-node DD, else x (rectsolver.py:102-109)
NN_RECT_CASES = [
    (12, 16, 0.1, 0.1, 0.0, "DDNN", ()),              # NN along y, DD sweep
    (20, 33, 0.05, 0.04, -3.0, "DDNN", ("west",)),    # + half-cell west end on the sweep
    (9, 64, 1.0 / 64, 1.0 / 64, 2.5, "IDNN", ("east",)),
    (16, 10, 0.1, 0.1, 0.0, "NNDD", ("south",)),      # y has a half-cell end -> NN along x
    (40, 24, 1.0 / 40, 1.0 / 24, -10.0, "NNDD", ("north", "south")),
    (130, 141, 1.0 / 141, 1.0 / 141, 0.0, "DDNN", ("east",)),
    # PP (real Fourier) transform axes
    (12, 16, 0.1, 0.1, 0.0, "DDPP", ()),
    (33, 64, 0.03, 1.0 / 64, -2.0, "NNPP", ("west",)),
    (18, 10, 0.1, 0.1, -1.0, "PPDD", ("south",)),
    (64, 256, 1.0 / 64, 1.0 / 256, 0.0, "IDPP", ("east",)),
]


def make_nn():
    """NN-transform rectangle solves and the reference's own test cross
    (bench.build_cross: Neumann flanks, half-cell Dirichlet arm ends) solved
    with its manufactured right-hand side, GMRES(50) to 1e-10."""
    from fftddm import bench as rbench
    out = {}
    rng = np.random.default_rng(11)
    for c, case in enumerate(NN_RECT_CASES):
        sub = rect(*case)
        pl = rectsolver.plan_rect(sub)
        f = rng.standard_normal(sub.size)
        out[f"nn_axis_{c}"] = np.array(pl.transform_axis)
        out[f"nn_f_{c}"] = f
        out[f"nn_p_{c}"] = rectsolver.solve_rect(pl, f).values
    for k_n in (2, 4, 8, 16):
        for kappa in (0.0, -3.0):
            case = rbench.build_cross(k_n=k_n, kappa=kappa)
            rhs = rbench.rhs_fields(case)
            fields, rep = ddm.ddm_solve(case.composite, rhs, krylov.GmresConfig(m=50, tol=1e-10))
            key = f"{k_n}_{int(-kappa)}"
            out[f"x_iters_{key}"] = np.array(rep.iterations)
            out[f"x_hist_{key}"] = np.asarray(rep.residual_history)
            for sub in case.composite.subdomains:
                out[f"x_f_{key}_{sub.id}"] = rhs[sub.id].values
                out[f"x_p_{key}_{sub.id}"] = fields[sub.id].values
    # comparison preconditioners (krylov.py:179-186) and the fixed-point
    # iteration (krylov.py:198-235) on the BASELINE cross geometry at N = 15
    comp, f, _, _ = configs.build_cross_case("c0", api=API, N=15)
    for pre in ("identity", "jacobi", "fft"):
        fields, rep = ddm.ddm_solve(comp, f, krylov.GmresConfig(m=50, tol=1e-10, preconditioner=pre))
        out[f"pre_iters_{pre}"] = np.array(rep.iterations)
        for sid, fld in fields.items():
            out[f"pre_p_{pre}_{sid}"] = fld.values
    op = ddm.build_schur_operator(comp)
    nbs = [nb for nb in op.neighbors]
    fp = f[op.coupled_id].copy()
    for nb in nbs:
        q = rectsolver.solve_rect(nb.plan, f[nb.plan.subdomain.id]).values
        fp = fp - nb.to_center.apply(q)
    out["fp_rhs"] = fp
    pc, rep = krylov.fixed_point(op, geometry.GridField(op.coupled_id, fp), max_iters=60, tol=1e-10)
    out["fp_iters"] = np.array(rep.iterations)
    out["fp_conv"] = np.array(rep.converged)
    out["fp_hist"] = np.asarray(rep.residual_history)
    out["fp_p"] = pc.values
    np.savez_compressed(os.path.join(HERE, "nn.npz"), **out)
    print("nn.npz written")


# periodic sweep axes (x periodic, transform along y): the Sherman-Morrison
# cyclic solve (rectsolver.py:136-153,202-205), m even
CYC_RECT_CASES = [
    (4, 3, 1.0, 1.0, 0.0, "PPDD", ()),
    (2, 5, 0.5, 0.25, 0.0, "PPDD", ()),              # two rows: doubled coupling
    (16, 12, 0.1, 0.1, 0.0, "PPDD", ()),
    (24, 16, 0.1, 0.1, -1.0, "PPNN", ()),
    (20, 12, 0.1, 0.1, -1.0, "PPPP", ()),
    (130, 141, 1.0 / 130, 1.0 / 141, -2.0, "PPDD", ()),
    (256, 63, 1.0 / 256, 1.0 / 64, 0.0, "PPDD", ()),  # many carry blocks
    (64, 255, 1.0 / 64, 1.0 / 256, 0.0, "PPDD", ()),  # an FFT length on the dense solve
]
# pin_mean: singular all-Neumann / periodic operators, mean-zero right-hand sides
PIN_RECT_CASES = [
    (3, 3, 1.0, 1.0, 0.0, "NNNN", ()),
    (8, 6, 0.1, 0.2, 0.0, "NNNN", ()),
    (6, 8, 0.1, 0.1, 0.0, "PPPP", ()),
    (16, 12, 0.1, 0.1, 0.0, "PPNN", ()),
    (12, 10, 0.1, 0.1, 0.0, "NNPP", ()),
    (40, 33, 1.0 / 40, 1.0 / 33, 0.0, "NNNN", ()),
]


def make_cyclic():
    """Periodic-sweep and pin_mean rectangle solves by the reference."""
    out = {}
    rng = np.random.default_rng(21)
    for c, case in enumerate(CYC_RECT_CASES):
        sub = rect(*case)
        pl = rectsolver.plan_rect(sub)
        assert pl.x_solver_kind == "cyclic"
        f = rng.standard_normal(sub.size)
        out[f"cyc_f_{c}"] = f
        out[f"cyc_p_{c}"] = rectsolver.solve_rect(pl, f).values
    for c, case in enumerate(PIN_RECT_CASES):
        sub = rect(*case)
        pl = rectsolver.plan_rect(sub, pin_mean=True)
        f = rng.standard_normal(sub.size)
        f -= f.mean()
        out[f"pin_modes_{c}"] = np.asarray(pl.singular_modes, dtype=np.int64)
        out[f"pin_f_{c}"] = f
        out[f"pin_p_{c}"] = rectsolver.solve_rect(pl, f).values
    np.savez_compressed(os.path.join(HERE, "cyclic.npz"), **out)
    print("cyclic.npz written")


def make_acceptance():
    """The reference's acceptance gates C3-C5 (tests/test_acceptance.py:78-128)
    run by the reference on its own cross: C3 node-error sup norms at k_n = 4..64
    (default GmresConfig), C4 fft / identity iteration counts at k_n = 16
    (m = 80, tol 1e-7, 25 restarts), C5 iteration counts at k_n = 8..128
    (m = 80, tol 1e-7).  Also checks that configs.reference_cross_case
    reproduces the reference's bench.rhs_fields / exact_fields bitwise."""
    from fftddm import bench
    from fftddm.errors import ConvergenceError
    from fftddm.geometry import GridField
    out = {}
    for kn in (4, 8, 16, 32, 64):
        case = bench.build_cross(k_n=kn)
        comp, f, exact = configs.reference_cross_case(kn, api=API)
        ref_f = bench.rhs_fields(case)
        ref_x = bench.exact_fields(case)
        for sid in f:
            assert np.array_equal(f[sid], ref_f[sid].values), ("rhs", kn, sid)
            assert np.array_equal(exact[sid], ref_x[sid].values), ("exact", kn, sid)
        t0 = time.perf_counter()
        fields, rep = bench.solve_case(case)
        linf, l2 = bench.error_norms(case, fields)
        out[f"c3_linf_{kn}"] = linf
        out[f"c3_l2_{kn}"] = l2
        out[f"c3_iters_{kn}"] = rep.iterations
        print("C3", kn, linf, rep.iterations, time.perf_counter() - t0, flush=True)
    case = bench.build_cross(k_n=16)
    op = ddm.build_schur_operator(case.composite)
    f = bench.rhs_fields(case)
    f_prime = f[op.coupled_id].values.copy()
    for nb in op.neighbors:
        f_prime -= nb.to_center.apply(rectsolver.solve_rect(nb.plan, f[nb.plan.subdomain.id]).values)
    rhs = GridField(op.coupled_id, f_prime)
    for mode in ("fft", "identity"):
        cfg = krylov.GmresConfig(m=80, tol=1e-7, max_restarts=25, preconditioner=mode)
        try:
            _, rep = krylov.solve_coupled(op, rhs, cfg)
            out[f"c4_iters_{mode}"] = rep.iterations
            out[f"c4_conv_{mode}"] = 1
        except ConvergenceError as exc:
            out[f"c4_iters_{mode}"] = exc.report.iterations
            out[f"c4_conv_{mode}"] = 0
        print("C4", mode, out[f"c4_iters_{mode}"], flush=True)
    rows = bench.run_scaling([8, 16, 32, 64, 128], tol_list=(1e-7,), m=80)
    for r in rows:
        out[f"c5_iters_{r['k_n']}"] = r["iterations"]
    out["c5_exponent"] = rows[0]["fitted_exponent"]
    print("C5", {r["k_n"]: r["iterations"] for r in rows}, rows[0]["fitted_exponent"], flush=True)
    np.savez_compressed(os.path.join(HERE, "acceptance.npz"), **out)
    print("acceptance.npz written")


if __name__ == "__main__":
    for what in sys.argv[1:] or ["small", "c0", "c1"]:
        if what == "small":
            make_small()
        elif what == "nn":
            make_nn()
        elif what == "cyclic":
            make_cyclic()
        elif what == "acceptance":
            make_acceptance()
        elif what == "c1":
            make_c1()
        else:
            solve_cross(what, full=(what == "c0"))
