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

_K = {"D": BoundaryKind.DIRICHLET, "N": BoundaryKind.NEUMANN, "I": BoundaryKind.INTERFACE,
      "P": BoundaryKind.PERIODIC}


def make(case, sid=0):
    m, n, dx, dy, kappa, bc, half = case
    edge_bc = {e: _K[c] for e, c in zip(("west", "east", "south", "north"), bc)}
    return RectSubdomain(id=sid, origin=(0.0, 0.0), m=m, n=n, dx=dx, dy=dy, edge_bc=edge_bc,
                         kappa=kappa, half_cell_dirichlet=frozenset(half))
