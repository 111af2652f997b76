"""The reference's acceptance gates C3-C5 (reference tests/test_acceptance.py:
78-128) through the GPU path, on the reference's own cross (its bench.py
build_cross: Neumann flanks, half-cell Dirichlet arm ends, NN transform axes)
with its manufactured problem (configs.reference_cross_case, checked bitwise
against the reference's rhs_fields / exact_fields by make_golden.py
acceptance).  Beyond the reference's own thresholds, the iteration counts
must equal the reference run's and the node errors match it to 1e-6."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2509_23180_b200 import configs, ddm, krylov, rectsolver  # noqa: E402
from paper_2509_23180_b200.errors import ConvergenceError  # noqa: E402
from paper_2509_23180_b200.geometry import GridField  # noqa: E402


def _linf(fields, exact):
    return max(float(np.abs(np.asarray(fields[s].values if not hasattr(fields[s].values, "cpu")
                                           else fields[s].values.cpu().numpy()) - exact[s]).max())
               for s in exact)


def test_criterion_3_second_order_convergence():
    """run_convergence([4, 8, 16, 32, 64]) with the default GmresConfig
    (m = 80, tol 1e-10): last two observed orders in [1.9, 2.1]."""
    g = load_golden("acceptance")
    errs = []
    for kn in (4, 8, 16, 32, 64):
        comp, f, exact = configs.reference_cross_case(kn)
        fields, rep = ddm.ddm_solve(comp, f)
        assert rep.iterations == int(g[f"c3_iters_{kn}"]), kn
        linf = _linf(fields, exact)
        assert linf == pytest.approx(float(g[f"c3_linf_{kn}"]), rel=1e-6), kn
        errs.append(linf)
    orders = [np.log2(errs[i - 1] / errs[i]) for i in (3, 4)]
    assert all(1.9 <= o <= 2.1 for o in orders), orders


def test_criterion_4_preconditioner_benefit():
    """k_n = 16, GMRES(80) to 1e-7 with at most 25 restarts on the coupled
    system: the FFT preconditioner needs at most 1/7 of the identity's
    iterations (the identity run hits its cap like the reference's)."""
    g = load_golden("acceptance")
    comp, f, _ = configs.reference_cross_case(16)
    op = ddm.build_schur_operator(comp)
    f_prime = np.array(f[op.coupled_id], dtype=float)
    for nb in op.neighbors:
        q = rectsolver.solve_rect(nb.plan, f[nb.plan.subdomain.id]).values
        q = q.cpu().numpy() if hasattr(q, "cpu") else np.asarray(q)
        f_prime -= nb.to_center.apply(q)
    rhs = GridField(op.coupled_id, f_prime)
    counts = {}
    for mode in ("fft", "identity"):
        cfg = krylov.GmresConfig(m=80, tol=1e-7, max_restarts=25, preconditioner=mode)
        try:
            _, rep = krylov.solve_coupled(op, rhs, cfg)
            counts[mode] = rep.iterations
        except ConvergenceError as exc:
            counts[mode] = exc.report.iterations
        assert counts[mode] == int(g[f"c4_iters_{mode}"]), mode
    assert counts["fft"] <= counts["identity"] / 7.0, counts


def test_criterion_5_iteration_scaling():
    """run_scaling([8 .. 128], tol 1e-7, m = 80): fitted exponent of
    iterations vs k_n in [0.3, 0.7], counts equal to the reference's."""
    g = load_golden("acceptance")
    kns, iters = [8, 16, 32, 64, 128], []
    for kn in kns:
        comp, f, _ = configs.reference_cross_case(kn)
        _, rep = ddm.ddm_solve(comp, f, krylov.GmresConfig(m=80, tol=1e-7))
        iters.append(rep.iterations)
        assert rep.iterations == int(g[f"c5_iters_{kn}"]), kn
    expo = float(np.polyfit(np.log(kns), np.log(iters), 1)[0])
    assert 0.3 <= expo <= 0.7, expo
    assert expo == pytest.approx(float(g["c5_exponent"]), abs=1e-12)
