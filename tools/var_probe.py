import sys, time, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2509_23180_b200 import configs, ddm, krylov, _native
import paper_2509_23180_b200.ddm as D
comp, f, exact, meta = configs.build_cross_case(sys.argv[1] if len(sys.argv) > 1 else "c3")
fd = {k: torch.as_tensor(v, device="cuda") for k, v in f.items()}
cfg = krylov.GmresConfig(m=50, tol=1e-10)
orig_build = D.build_schur_operator
def timed_build(*a, **k):
    t0 = time.perf_counter(); r = orig_build(*a, **k); torch.cuda.synchronize(); print(f"  build {time.perf_counter()-t0:.3f}", flush=True); return r
D.build_schur_operator = timed_build
lib = _native.lib()
orig = lib.fd_ddm_solve
t_native = [0.0]
def wrapped(*a):
    t0 = time.perf_counter(); r = orig(*a); print(f"  native {time.perf_counter()-t0:.3f}", flush=True); return r
lib.fd_ddm_solve = wrapped
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
for i in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    fields, rep = ddm.ddm_solve(comp, fd, cfg)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"call {i}: {t1-t0:.3f} s, gmres {rep.wall_time:.3f}", flush=True)
    del fields
