"""Per-kernel times of the split solve (FD_SPLIT=1 FD_SPLIT_TIMING=1): a few c1 applies."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_23180_b200 import configs, rectsolver
rng = np.random.default_rng(1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1023
subs = configs.batch_rects(n, 5, 0.0)
plans = [rectsolver.plan_rect(s) for s in subs]
sets = [[torch.as_tensor(rng.uniform(-1, 1, s.size), device="cuda") for s in subs] for _ in range(8)]
outs = [[torch.empty_like(x) for x in fs] for fs in sets]
for i in range(12):
    rectsolver.solve_rect_batched(plans, sets[i % 8], outs[i % 8])
torch.cuda.synchronize()
