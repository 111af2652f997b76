"""K3 bring-up: rectangle solves at n = 1023 against the oracle (several m,
batches of different m, kappa) and the c1 apply time with 8 rotating buffer
sets (CUDA events)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import fftddm_oracle as O  # noqa: E402
from paper_2509_23180_b200 import configs, rectsolver  # noqa: E402
from paper_2509_23180_b200.geometry import BoundaryKind, RectSubdomain  # noqa: E402

D = BoundaryKind.DIRICHLET
rng = np.random.default_rng(1)


def sub(m, n, kappa):
    bc = {e: D for e in ("west", "east", "south", "north")}
    return RectSubdomain(id=0, origin=(0.0, 0.0), m=m, n=n, dx=1 / n, dy=1 / n, edge_bc=bc, kappa=kappa)


worst = 0.0
for ms, kappa in [((1,), 0.0), ((2,), 0.0), ((3,), -10.0), ((17,), 0.0), ((149,), -10.0), ((1023,), 0.0),
                  ((1185,), 7.0), ((5, 300, 1023), -100.0), ((1023,) * 5, -10.0)]:
    subs = [sub(m, 1023, kappa) for m in ms]
    f = [rng.uniform(-1, 1, s.size) for s in subs]
    plans = [rectsolver.plan_rect(s) for s in subs]
    outs = rectsolver.solve_rect_batched(plans, f)
    errs = []
    for s, fi, o in zip(subs, f, outs):
        ref = O.solve(O.plan(s), fi)
        v = o.cpu().numpy() if hasattr(o, "cpu") else np.asarray(o)
        errs.append(np.linalg.norm(v - ref) / np.linalg.norm(ref))
    worst = max(worst, max(errs))
    print(f"m={ms} kappa={kappa}: rel err max {max(errs):.3e}", flush=True)
print(f"WORST {worst:.3e}")

subs = configs.batch_rects(1023, 5, 0.0)
plans = [rectsolver.plan_rect(s) for s in subs]
sets = [[torch.as_tensor(rng.uniform(-1, 1, s.size), device="cuda") for s in subs] for _ in range(8)]
outs = [[torch.empty_like(x) for x in fs] for fs in sets]
for i in range(5):
    rectsolver.solve_rect_batched(plans, sets[i % 8], outs[i % 8])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 200
e0.record()
for i in range(R):
    rectsolver.solve_rect_batched(plans, sets[i % 8], outs[i % 8])
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / R * 1e3
print(f"c1 apply: {us:.1f} us  ({32 * 5 * 1023 * 1023 / us / 1e3:.0f} GB/s algorithmic)")
