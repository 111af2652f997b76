"""The C-ABI library loads, exports every symbol include/fftddm_b200.h declares,
and its host-side plan tables match the reference's factorisation.  No GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2509_23180_b200 import _native, build
from rects import RECT_CASES, make

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "fftddm_b200.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _native.lib()


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fd_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_binding():
    assert declared() == sorted(_native.EXPORTS)


def test_exports(lib):
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.fd_version() >= 100


def test_symbols_visible_in_dynsym(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    missing = [n for n in declared() if n not in syms]
    assert not missing, missing


def _host_tables(lib, m, n, dx, dy, kappa, mw, me):
    beta = np.empty((m, n))
    lower = np.empty((m, n))
    st = lib.fd_factor_tables_host(m, n, dx, dy, kappa, mw, me,
                                   beta.ctypes.data_as(_native.DP), lower.ctypes.data_as(_native.DP))
    return st, beta, lower


@pytest.mark.parametrize("c", range(len(RECT_CASES)))
def test_factor_tables_match_reference(lib, golden_small, c):
    if f"rect_beta_{c}" not in golden_small:
        pytest.skip("large case: factors not stored")
    sub = make(RECT_CASES[c])
    st, beta, lower = _host_tables(lib, sub.m, sub.n, sub.dx, sub.dy, sub.kappa,
                                   sub.end_modifier("west"), sub.end_modifier("east"))
    assert st == 0
    ref_b, ref_l = golden_small[f"rect_beta_{c}"], golden_small[f"rect_lower_{c}"]
    # eigenvalues come from libm cos vs numpy's SIMD cos: allow 2 ulp
    np.testing.assert_allclose(beta, ref_b, rtol=5e-16, atol=0)
    np.testing.assert_allclose(lower, ref_l, rtol=5e-16, atol=0)


def test_factor_tables_large_compressed(lib):
    """Compressed tables (fixed-point prefix + constant) reproduce the full
    sequential recurrence at config-2/3 sizes (oracle restatement)."""
    import fftddm_oracle as O
    m, n = 4095, 63
    dx = dy = 1.0 / 4095
    st, beta, lower = _host_tables(lib, m, n, dx, dy, -100.0, 0.0, 0.0)
    assert st == 0
    lam = O.eigenvalues_dd(n, 1 / dy ** 2, 1 / dx ** 2, -100.0)
    b, l, bad = O.factor_tridiag(np.tile(lam, (m, 1)), 1 / dx ** 2, 1e-13 * max(abs(lam).max(), 1 / dx ** 2))
    np.testing.assert_allclose(beta, b, rtol=5e-16, atol=0)
    np.testing.assert_allclose(lower, l, rtol=5e-16, atol=0)


def test_singular_reported(lib):
    # all-Neumann sweep with kappa = 0 and the zero DD mode cannot vanish; force a
    # zero pivot with a 1 x 1 grid whose diagonal is exactly 0: kappa = 4
    st, _, _ = _host_tables(lib, 1, 1, 1.0, 1.0, 4.0, 0.0, 0.0)
    assert st == _native.FD_ERR_SINGULAR
    assert b"singular" in lib.fd_last_error()


def test_errors_map_to_reference_classes():
    from paper_2509_23180_b200.errors import SingularOperatorError, ValidationError
    with pytest.raises(SingularOperatorError):
        _native.lib().fd_last_error  # noqa: B018
        _native.check(_native.FD_ERR_SINGULAR)
    with pytest.raises(ValidationError):
        _native.check(_native.FD_ERR_VALIDATION)
    with pytest.raises(NotImplementedError):
        _native.check(_native.FD_ERR_UNSUPPORTED)


def test_transform_kind(lib):
    """GPU transform availability per length (drives the axis choice)."""
    assert [lib.fd_transform_kind(n) for n in (255, 511, 1023, 2047, 4095)] == [1] * 5
    assert [lib.fd_transform_kind(n) for n in (1, 141, 1000, 1024, 1025, 1500, 2048)] == [0] * 7
    # any other length: the separate Stockham / Bluestein passes (kSep)
    assert [lib.fd_transform_kind(n) for n in (2049, 3000, 8191, 16383, 65535)] == [2] * 5
    assert [lib.fd_transform_kind(n) for n in (0, 65536)] == [-1] * 2


@pytest.mark.parametrize("m,n,bc,half,axis", [
    (1023, 1023, "DDDD", (), "y"),          # c1: the reference's choice
    (16383, 4095, "DDDD", (), "y"),         # c4 west/east arm
    (4095, 16383, "DDDD", (), "x"),         # c4 south/north arm: no 16384-point transform -> x
    (255, 127, "DDDD", ("south",), "x"),    # y half-cell -> x, as the reference
    (9, 31, "IDDD", ("east",), "y"),        # sweep-axis modifiers only
    (40, 3000, "DDDD", (), "x"),            # n without a GPU length, m with one -> x
    (40, 1500, "DDDD", (), "y"),            # n <= 2048: dense transform along y, as the reference
    (3000, 3000, "DDDD", (), "y"),          # neither: the reference's y (plan creation reports it)
])
def test_gpu_axis_choice(lib, m, n, bc, half, axis):
    from paper_2509_23180_b200.rectsolver import _gpu_axis
    assert _gpu_axis(make((m, n, 1.0 / n, 1.0 / n, 0.0, bc, half))) == axis


def test_gpu_axis_unsupported(lib):
    from paper_2509_23180_b200._native import UnsupportedError
    from paper_2509_23180_b200.rectsolver import _gpu_axis
    with pytest.raises(UnsupportedError):
        _gpu_axis(make((12, 9, 1.0, 1.0, 0.0, "DDDD", ("west", "south"))))


def test_interface_line_descriptors():
    """Interface-only variant: line geometry of each arm of the BASELINE cross
    (host logic, no GPU): the line runs along the interface, the sweep across
    it, and the interface row is the sweep's first or last row."""
    from paper_2509_23180_b200 import configs, ddm
    comp = configs.cross_composite(15, arm=40, kappa=-2.0)
    centre = comp.subdomain(0)
    seen = {}
    for iface in comp.interfaces_of(0):
        other = iface.other_side(0)[0]
        sub = comp.subdomain(other)
        edge = iface.side_a[1] if iface.side_a[0] == other else iface.side_b[1]
        to_c = ddm.make_coupling(comp, iface, other)
        from_c = ddm.make_coupling(comp, iface, 0)
        L, M, dl, ds, mlo, mhi, end, pin, pout = ddm._steklov_line(sub, edge, to_c, from_c)
        assert L == 15 and M == 40 and end == (1 if edge in ("east", "north") else 0)
        assert sorted(pin.tolist()) == list(range(15)) and sorted(pout.tolist()) == list(range(15))
        assert mlo == 0.0 and mhi == 0.0 and dl == pytest.approx(15.0 ** 2) and ds == pytest.approx(15.0 ** 2)
        seen[edge] = True
    assert sorted(seen) == ["east", "north", "south", "west"]
    # a half-cell end on the line's own axis disqualifies the line
    ref = configs.reference_cross(4)
    for iface in ref.interfaces_of(0):
        other = iface.other_side(0)[0]
        sub = ref.subdomain(other)
        edge = iface.side_a[1] if iface.side_a[0] == other else iface.side_b[1]
        assert ddm._steklov_line(sub, edge, ddm.make_coupling(ref, iface, other),
                                 ddm.make_coupling(ref, iface, 0)) is None   # NN flanks along the line
