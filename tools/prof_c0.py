"""One c0 solve (for ncu captures of the dense-path kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, ddm, krylov  # noqa: E402

comp, f, _, _ = configs.build_cross_case("c0")
fd = {k: torch.as_tensor(v, device="cuda") for k, v in f.items()}
for _ in range(2):
    ddm.ddm_solve(comp, fd, krylov.GmresConfig(m=50, tol=1e-10))
torch.cuda.synchronize()
print("ok")
