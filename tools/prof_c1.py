"""Short c1 run for Nsight Compute: W warm-up + K batched applies (5 x 1023^2)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, rectsolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1023)
ap.add_argument("--count", type=int, default=5)
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
subs = configs.batch_rects(args.n, args.count, 0.0)
plans = [rectsolver.plan_rect(s) for s in subs]
rng = np.random.default_rng(0)
f = [torch.as_tensor(rng.uniform(-1, 1, s.size), device="cuda") for s in subs]
out = [torch.empty_like(x) for x in f]
for _ in range(args.steps):
    rectsolver.solve_rect_batched(plans, f, out)
torch.cuda.synchronize()
print("ok")
