"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every production kernel family at small sizes -- the FFT-path persistent solve
(n = 255, ragged batch), the dense-path solve (n = 141), the transposed axis,
the Schur operator + low-sync GMRES on a small cross (N = 15, 31 with m = 80),
the interface-only variant and device assembly."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_23180_b200 import configs, ddm, krylov, rectsolver  # noqa: E402
from paper_2509_23180_b200.geometry import BoundaryKind, RectSubdomain  # noqa: E402

D = BoundaryKind.DIRICHLET
bc = {e: D for e in ("west", "east", "south", "north")}
rng = np.random.default_rng(0)


def sub(m, n, kappa=0.0):
    return RectSubdomain(id=0, origin=(0.0, 0.0), m=m, n=n, dx=1 / n, dy=1 / n, edge_bc=bc, kappa=kappa)


subs = [sub(m, 255, -3.0) for m in (3, 17, 40)]
outs = rectsolver.solve_rect_batched([rectsolver.plan_rect(s) for s in subs], [rng.uniform(-1, 1, s.size) for s in subs])
s = sub(20, 141, -1.0)
rectsolver.solve_rect(rectsolver.plan_rect(s), rng.uniform(-1, 1, s.size))
s = sub(30, 2100, 0.0)   # transform along x
rectsolver.solve_rect(rectsolver.plan_rect(s), rng.uniform(-1, 1, s.size))
for N, m in ((15, 50), (31, 80)):
    comp, f, _, _ = configs.build_cross_case("c0", N=N)
    ddm.ddm_solve(comp, f, krylov.GmresConfig(m=m, tol=1e-10))
comp, f, _, _ = configs.build_cross_case("c3", N=63)
ddm.ddm_solve(comp, f, krylov.GmresConfig(m=50, tol=1e-10), interface_only=True)
configs.build_cross_case("c0", N=31, device=True)
torch.cuda.synchronize()
print("sanitize workload ok")
