"""Timing of the dense periodic-table path on transforms longer than 1024
(DD n=1500, NN n=2048, PP n=2048; m = n), one rectangle, device-resident."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from rects import make  # noqa: E402
from paper_2509_23180_b200 import rectsolver  # noqa: E402
for bc, n in [("DDDD", 1500), ("DDNN", 2048), ("DDPP", 2048), ("DDDD", 1023)]:
    sub = make((n, n, 1.0 / n, 1.0 / n, -1.0, bc, ()))
    pl = rectsolver.plan_rect(sub)
    f = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, sub.size), device="cuda")
    out = torch.empty_like(f)
    for _ in range(3):
        rectsolver.solve_rect_batched([pl], [f], [out])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        rectsolver.solve_rect_batched([pl], [f], [out])
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{bc} n={n}: {dt*1e3:.3f} ms per {n}x{n} solve, {n*n/dt/1e9:.2f} Gpts/s, axis {pl.transform_axis}")
