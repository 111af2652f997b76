import sys; sys.path.insert(0, "/root/repo")
from paper_2509_23180_b200 import configs, ddm, krylov
for N, tol in ((3000, 1e-10), (3000, 1e-12), (2999, 1e-10), (3001, 1e-10), (2500, 1e-10)):
    comp, fd, exd, _ = configs.build_cross_case("c0", N=N, device=True)
    fields, rep = ddm.ddm_solve(comp, fd, krylov.GmresConfig(m=50, tol=tol))
    print(N, tol, rep.iterations, configs.rel_l2_device(fields, exd), flush=True)
