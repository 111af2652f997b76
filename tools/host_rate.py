"""Host enqueue cost of the batched c1 apply vs its GPU time."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, rectsolver
subs = configs.batch_rects(1023, 5, 0.0)
plans = [rectsolver.plan_rect(s) for s in subs]
rng = np.random.default_rng(0)
f = [torch.as_tensor(rng.uniform(-1, 1, s.size), device="cuda") for s in subs]
out = [torch.empty_like(x) for x in f]
for _ in range(5):
    rectsolver.solve_rect_batched(plans, f, out)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N):
    rectsolver.solve_rect_batched(plans, f, out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6 * (t1 - t0) / N:.1f} us/apply, wall {1e6 * (t2 - t0) / N:.1f} us/apply")
