"""Where the numpy-in / numpy-out time of a c2 solve goes (per phase)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, ddm, krylov, _fields
comp, f, exact, meta = configs.build_cross_case("c2")
cfg = krylov.GmresConfig(m=50, tol=1e-10)
fd = {k: torch.as_tensor(v, device="cuda") for k, v in f.items()}
ddm.ddm_solve(comp, fd, cfg); torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); ddm.ddm_solve(comp, f, cfg); t1 = time.perf_counter()
    t2 = time.perf_counter(); ddm.ddm_solve(comp, fd, cfg); torch.cuda.synchronize(); t3 = time.perf_counter()
    a = time.perf_counter(); vs = [_fields.to_device(v, v.size)[0] for v in f.values()]; torch.cuda.synchronize(); b = time.perf_counter()
    outs = [_fields.like_input(v, True) for v in vs]; c = time.perf_counter()
    print(f"numpy path {t1-t0:.3f} s, device path {t3-t2:.3f} s, H2D all {b-a:.3f} s, D2H all {c-b:.3f} s", flush=True)
