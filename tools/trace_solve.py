"""Kernel/API trace of one ddm_solve (torch.profiler / CUPTI).

    python tools/trace_solve.py [c0|c2|c3] [--N n]

Prints the top kernels and CUDA runtime calls by total time, the summed
kernel time vs the wall time, and writes a chrome trace to gpurun_out/.
"""
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, ddm, krylov  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "c0"
kw = {}
if "--N" in sys.argv:
    kw["N"] = int(sys.argv[sys.argv.index("--N") + 1])
comp, f, exact, meta = configs.build_cross_case(name, **kw)
fd = {k: torch.as_tensor(v, device="cuda") for k, v in f.items()}
cfg = krylov.GmresConfig(m=50, tol=1e-10)
ddm.ddm_solve(comp, fd, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    fields, rep = ddm.ddm_solve(comp, fd, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
print(f"{name}: wall {wall*1e3:.2f} ms, iterations {rep.iterations}, gmres {rep.wall_time*1e3:.2f} ms")
ka = prof.key_averages()
print(ka.table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
print(ka.table(sort_by="cpu_time_total", row_limit=25, max_name_column_width=70))
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(f"gpurun_out/trace_{name}.json")
