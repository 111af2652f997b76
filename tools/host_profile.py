"""cProfile of one ddm_solve (host-side setup cost: plans, couplings, shim)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, ddm, krylov  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
comp, f, exact, meta = configs.build_cross_case(name)
fd = {k: torch.as_tensor(v, device="cuda") for k, v in f.items()}
cfg = krylov.GmresConfig(m=50, tol=1e-10)
ddm.ddm_solve(comp, fd, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
ddm.ddm_solve(comp, fd, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
