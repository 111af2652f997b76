"""Rectangle cases mirrored from tests/golden/make_golden.py RECT_CASES."""
from paper_2509_23180_b200.geometry import BoundaryKind, RectSubdomain

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

# periodic sweep axes (make_golden.py CYC_RECT_CASES) and pin_mean cases (PIN_RECT_CASES)
CYC_RECT_CASES = [
    (4, 3, 1.0, 1.0, 0.0, "PPDD", ()),
    (2, 5, 0.5, 0.25, 0.0, "PPDD", ()),
    (16, 12, 0.1, 0.1, 0.0, "PPDD", ()),
    (24, 16, 0.1, 0.1, -1.0, "PPNN", ()),
    (20, 12, 0.1, 0.1, -1.0, "PPPP", ()),
    (130, 141, 1.0 / 130, 1.0 / 141, -2.0, "PPDD", ()),
    (256, 63, 1.0 / 256, 1.0 / 64, 0.0, "PPDD", ()),
    (64, 255, 1.0 / 64, 1.0 / 256, 0.0, "PPDD", ()),
]
PIN_RECT_CASES = [
    (3, 3, 1.0, 1.0, 0.0, "NNNN", ()),
    (8, 6, 0.1, 0.2, 0.0, "NNNN", ()),
    (6, 8, 0.1, 0.1, 0.0, "PPPP", ()),
    (16, 12, 0.1, 0.1, 0.0, "PPNN", ()),
    (12, 10, 0.1, 0.1, 0.0, "NNPP", ()),
    (40, 33, 1.0 / 40, 1.0 / 33, 0.0, "NNNN", ()),
]


def pair_cases(max_mn=5):
    """All transform/sweep pair combinations on small grids, PP counts even and
    kappa negative where the operator would be singular (the reference's
    test_rectsolver.pair_cases rule)."""
    for x_pair in ("DD", "NN", "PP"):
        for y_pair in ("DD", "NN", "PP"):
            for m in range(1, max_mn + 1):
                for n in range(1, max_mn + 1):
                    if (x_pair == "PP" and m % 2) or (y_pair == "PP" and n % 2):
                        continue
                    kappa = -1.0 if "DD" not in (x_pair, y_pair) else 0.0
                    yield x_pair, y_pair, m, n, kappa


def pair_rect(x_pair, y_pair, m, n, kappa, sid=0):
    bc = x_pair[0] * 2 + y_pair[0] * 2
    return make((m, n, 0.5, 0.25, kappa, bc, ()), sid)


_K = {"D": BoundaryKind.DIRICHLET, "N": BoundaryKind.NEUMANN, "I": BoundaryKind.INTERFACE,
      "P": BoundaryKind.PERIODIC}


def make(case, sid=0):
    m, n, dx, dy, kappa, bc, half = case
    edge_bc = {e: _K[c] for e, c in zip(("west", "east", "south", "north"), bc)}
    return RectSubdomain(id=sid, origin=(0.0, 0.0), m=m, n=n, dx=dx, dy=dy, edge_bc=edge_bc,
                         kappa=kappa, half_cell_dirichlet=frozenset(half))
