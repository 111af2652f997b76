"""Pin the CPU oracle (oracle/fftddm_oracle.py) to fixtures written by the real
reference (tests/golden/make_golden.py) and to the reference's own
known-answer tests.  CPU only."""
import numpy as np
import pytest

import fftddm_oracle as O
from conftest import load_golden, rel
from paper_2509_23180_b200 import configs
from rects import RECT_CASES, make


class TestKnownAnswers:
    def test_eigenvalues_dd(self):
        # test_transforms.py:20-27
        np.testing.assert_allclose(O.eigenvalues_dd(1, 1.0, 1.0), [-4.0], atol=1e-15)
        np.testing.assert_allclose(sorted(O.eigenvalues_dd(3, 1.0, 1.0)),
                                   sorted([-4 + np.sqrt(2), -4.0, -4 - np.sqrt(2)]))

    def test_apply_q_first_basis_vector(self):
        # test_transforms.py:64-68
        np.testing.assert_allclose(O.apply_q_dd(np.array([1.0, 0.0, 0.0])),
                                   [0.5, 1 / np.sqrt(2), 0.5], atol=1e-14)

    def test_thomas_example(self):
        # test_rectsolver.py:31-34: tridiag(1, -2, 1) x = e1
        beta, lower, bad = O.factor_tridiag(np.full((3, 1), -2.0), 1.0, 1e-13)
        x = O.tridiag_solve(beta, lower, 1.0, np.array([[1.0], [0.0], [0.0]]))
        np.testing.assert_allclose(x[:, 0], [-0.75, -0.5, -0.25])
        assert not bad.any()

    def test_one_by_one(self):
        # test_rectsolver.py:70-73: 1x1 DD with unit spacing -> -1/4
        sub = make((1, 1, 1.0, 1.0, 0.0, "DDDD", ()))
        assert O.solve(O.plan(sub), np.array([1.0]))[0] == pytest.approx(-0.25)

    def test_q_orthonormal(self):
        Q = O.apply_q_dd(np.eye(17))
        np.testing.assert_allclose(Q @ Q, np.eye(17), atol=1e-14)


class TestAgainstReferenceFixtures:
    @pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 8, 15, 31, 63, 64, 127, 141, 255, 511, 1023,
                                   2047, 4095])
    def test_dst(self, golden_small, n):
        out = O.apply_q_dd(golden_small[f"dst_in_{n}"])
        assert rel(out, golden_small[f"dst_out_{n}"]) < 1e-15
        lam = O.eigenvalues_dd(n, 2.5, 0.75, kappa=-0.5)
        np.testing.assert_array_equal(lam, golden_small[f"eig_{n}"])

    @pytest.mark.parametrize("c", range(len(RECT_CASES)))
    def test_rect(self, golden_small, c):
        sub = make(RECT_CASES[c])
        pl = O.plan(sub)
        if f"rect_beta_{c}" in golden_small:
            np.testing.assert_array_equal(pl.beta, golden_small[f"rect_beta_{c}"])
            np.testing.assert_array_equal(pl.lower, golden_small[f"rect_lower_{c}"])
        p = O.solve(pl, golden_small[f"rect_f_{c}"])
        np.testing.assert_array_equal(p, golden_small[f"rect_p_{c}"])
        np.testing.assert_array_equal(O.apply_operator(sub, golden_small[f"rect_f_{c}"]),
                                      golden_small[f"rect_Av_{c}"])

    @pytest.mark.parametrize("N", [4, 8, 15, 31])
    @pytest.mark.parametrize("kappa", [0.0, -100.0])
    def test_cross(self, golden_small, N, kappa):
        tag = f"{N}_{int(-kappa)}"
        comp = configs.cross_composite(N, kappa=kappa)
        op = O.Schur(comp)
        p = golden_small[f"x_p_{tag}"]
        np.testing.assert_array_equal(op.schur(p), golden_small[f"x_schur_{tag}"])
        np.testing.assert_array_equal(op.preconditioned(p), golden_small[f"x_pre_{tag}"])
        np.testing.assert_array_equal(op.unpreconditioned(p), golden_small[f"x_unpre_{tag}"])
        f, _ = configs.manufactured_rhs(comp, "sin_exp")
        fields, rep = O.ddm_solve(comp, f, m=50, tol=1e-10)
        assert rep.iterations == int(golden_small[f"x_iters_{tag}"])
        np.testing.assert_allclose(rep.residual_history, golden_small[f"x_hist_{tag}"],
                                   rtol=1e-9, atol=0)
        for sid in range(5):
            assert rel(fields[sid], golden_small[f"x_sol_{tag}_{sid}"]) < 1e-14

    def test_gmres_dense(self, golden_small):
        A, b = golden_small["gm_A"], golden_small["gm_b"]
        x, rep = O.gmres(lambda v: A @ v, b, m=7, tol=1e-12)
        assert rep.iterations == int(golden_small["gm_iters"])
        assert rel(x, golden_small["gm_x"]) < 1e-13

    def test_c0_full(self):
        g = load_golden("c0")
        comp, f, exact, meta = configs.build_cross_case("c0")
        fields, rep = O.ddm_solve(comp, f, m=50, tol=1e-10)
        assert rep.iterations == int(g["iterations"]) == 38
        for sid in range(5):
            assert rel(fields[sid], g[f"sol_{sid}"]) < 1e-13
        assert configs.rel_l2(fields, exact) == pytest.approx(float(g["rel_l2_exact"]), rel=1e-9)


NN_RECT_CASES = [
    (12, 16, 0.1, 0.1, 0.0, "DDNN", ()),
    (20, 33, 0.05, 0.04, -3.0, "DDNN", ("west",)),
    (9, 64, 1.0 / 64, 1.0 / 64, 2.5, "IDNN", ("east",)),
    (16, 10, 0.1, 0.1, 0.0, "NNDD", ("south",)),
    (40, 24, 1.0 / 40, 1.0 / 24, -10.0, "NNDD", ("north", "south")),
    (130, 141, 1.0 / 141, 1.0 / 141, 0.0, "DDNN", ("east",)),
    (12, 16, 0.1, 0.1, 0.0, "DDPP", ()),
    (33, 64, 0.03, 1.0 / 64, -2.0, "NNPP", ("west",)),
    (18, 10, 0.1, 0.1, -1.0, "PPDD", ("south",)),
    (64, 256, 1.0 / 64, 1.0 / 256, 0.0, "IDPP", ("east",)),
]


@pytest.fixture(scope="module")
def golden_nn():
    return load_golden("nn")


class TestNeumannTransformFixtures:
    """NN (shifted-cosine) transform axes and the reference's own test cross,
    against fixtures written by the reference (tests/golden/make_golden.py nn)."""

    @pytest.mark.parametrize("c", range(len(NN_RECT_CASES)))
    def test_rect(self, golden_nn, c):
        from rects import make
        sub = make(NN_RECT_CASES[c])
        pl = O.plan(sub)
        assert pl.axis == str(golden_nn[f"nn_axis_{c}"])
        p = O.solve(pl, golden_nn[f"nn_f_{c}"])
        ref = golden_nn[f"nn_p_{c}"]
        assert rel(p, ref) < 1e-13

    def test_nn_basis_orthonormal(self):
        for n in (1, 2, 5, 16):
            Q = O.apply_q("NN", np.eye(n))
            np.testing.assert_allclose(Q @ Q.T, np.eye(n), atol=1e-13)
            np.testing.assert_allclose(O.apply_qt("NN", O.apply_q("NN", np.eye(n))), np.eye(n), atol=1e-13)

    @pytest.mark.parametrize("k_n,kappa", [(2, 0.0), (4, -3.0), (8, 0.0)])
    def test_reference_cross(self, golden_nn, k_n, kappa):
        comp = configs.reference_cross(k_n, kappa=kappa)
        key = f"{k_n}_{int(-kappa)}"
        f = {s.id: golden_nn[f"x_f_{key}_{s.id}"] for s in comp.subdomains}
        fields, rep = O.ddm_solve(comp, f, m=50, tol=1e-10)
        assert rep.iterations == int(golden_nn[f"x_iters_{key}"])
        for s in comp.subdomains:
            assert rel(fields[s.id], golden_nn[f"x_p_{key}_{s.id}"]) < 1e-12


class TestPeriodicSweepFixtures:
    """Periodic sweep axes (Sherman-Morrison cyclic solve, rectsolver.py:136-153,
    202-205) and pin_mean minimum-norm modes (rectsolver.py:157-175,206-207),
    against fixtures written by the reference (make_golden.py cyclic)."""

    @pytest.mark.parametrize("c", range(8))
    def test_cyclic_rect(self, c):
        from rects import CYC_RECT_CASES
        g = load_golden("cyclic")
        pl = O.plan(make(CYC_RECT_CASES[c]))
        assert pl.cyclic
        np.testing.assert_array_equal(O.solve(pl, g[f"cyc_f_{c}"]), g[f"cyc_p_{c}"])

    @pytest.mark.parametrize("c", range(6))
    def test_pin_mean_rect(self, c):
        from rects import PIN_RECT_CASES
        g = load_golden("cyclic")
        sub = make(PIN_RECT_CASES[c])
        with pytest.raises(O.SingularOracleError):
            O.plan(sub)
        pl = O.plan(sub, pin_mean=True)
        assert list(pl.singular) == g[f"pin_modes_{c}"].tolist()
        p = O.solve(pl, g[f"pin_f_{c}"])
        np.testing.assert_array_equal(p, g[f"pin_p_{c}"])
        # the GPU shim's pseudo-inverse form of lstsq (rectsolver.plan_rect)
        for M in pl.singular_dense:
            f = np.random.default_rng(3).standard_normal(M.shape[0])
            f -= f.mean()
            a = np.linalg.lstsq(M, f, rcond=None)[0]
            b = np.linalg.pinv(M, rcond=np.finfo(float).eps * M.shape[0]) @ f
            assert np.abs(a - b).max() <= 1e-13 * max(np.abs(a).max(), 1.0)

    def test_pair_sweep_residual(self):
        """Every transform/sweep pair on small grids: A p = f with the oracle's
        own stencil (periodic wrap included)."""
        from rects import pair_cases, pair_rect
        rng = np.random.default_rng(5)
        for case in pair_cases(5):
            sub = pair_rect(*case)
            f = rng.standard_normal(sub.size)
            p = O.solve(O.plan(sub), f)
            r = O.apply_operator(sub, p) - f
            assert np.abs(r).max() <= 1e-10 * max(np.abs(f).max(), 1.0), case


def test_reference_cross_acceptance_goldens():
    """The oracle on the reference's own cross (configs.reference_cross_case,
    NN arms, half-cell ends) reproduces the reference's C3 run at k_n = 4, 8:
    same iteration counts, node errors to 1e-9 (pins the restated
    manufactured problem used by the GPU acceptance tests)."""
    import numpy as np
    from conftest import load_golden
    from paper_2509_23180_b200 import configs
    import fftddm_oracle as O
    g = load_golden("acceptance")
    for kn in (4, 8):
        comp, f, exact = configs.reference_cross_case(kn)
        fields, rep = O.ddm_solve(comp, f, m=80, tol=1e-10)
        assert rep.iterations == int(g[f"c3_iters_{kn}"])
        linf = max(float(np.abs(fields[s] - exact[s]).max()) for s in exact)
        assert abs(linf - float(g[f"c3_linf_{kn}"])) <= 1e-9 * float(g[f"c3_linf_{kn}"])
