"""End-to-end ddm_solve timing on the BASELINE cross configs (GPU).

    python tools/solve_timing.py [c0 c2 c3] [--reps R]

RHS resident on the device; timed region = ddm_solve (plan build, arm
pre-solves, GMRES to 1e-10, back-substitution), CUDA-synchronised, median of
R repetitions after one warm-up.  Prints one JSON line per config.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, ddm, krylov  # noqa: E402


def main():
    argv = sys.argv[1:]
    names = [a for i, a in enumerate(argv) if not a.startswith("--") and not (i and argv[i - 1] == "--reps")]
    names = names or ["c0", "c2", "c3"]
    reps = 5
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
    for name in names:
        if "--assemble" in sys.argv and name != "c3":
            # problem assembled on the device inside the timed region
            comp, fd, exact_d, meta = configs.build_cross_case(name, device=True)
            exact = None
        else:
            comp, f, exact, meta = configs.build_cross_case(name)
            fd = {k: torch.as_tensor(v, device="cuda") for k, v in f.items()}
            del f
            exact_d = None
        cfg = krylov.GmresConfig(m=50, tol=1e-10)
        kw = {"interface_only": True} if "--steklov" in sys.argv else {}
        fields, rep = ddm.ddm_solve(comp, fd, cfg, **kw)   # warm-up (module load, tables)
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if exact_d is not None:
                comp, fd, exact_d, meta = configs.build_cross_case(name, device=True)
            fields, rep = ddm.ddm_solve(comp, fd, cfg, **kw)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        wall = float(np.median(times))
        tag = (" interface-only" if kw else "") + (" +assembly" if exact_d is not None else "")
        out = {"config": name + tag, "points": meta["points"], "iterations": rep.iterations,
               "wall_s": wall, "mpts_per_s": meta["points"] / wall / 1e6,
               "gmres_wall_s": rep.wall_time, "all_s": [round(t, 4) for t in times], "us_per_iteration": rep.wall_time / max(rep.iterations, 1) * 1e6,
               "true_residual": rep.true_residual}
        if exact is not None:
            out["rel_l2_exact"] = configs.rel_l2(fields, exact)
        if exact_d is not None:
            out["rel_l2_exact"] = configs.rel_l2_device(fields, exact_d)
            out["timing"] = "device assembly of the manufactured problem + ddm_solve"
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
