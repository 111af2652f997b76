"""One c2 ddm_solve for a kernel launch list (ncu)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, ddm, krylov  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
comp, f, exact, meta = configs.build_cross_case(name)
fd = {k: torch.as_tensor(v, device="cuda") for k, v in f.items()}
fields, rep = ddm.ddm_solve(comp, fd, krylov.GmresConfig(m=50, tol=1e-10))
torch.cuda.synchronize()
print(rep.iterations, rep.wall_time)
