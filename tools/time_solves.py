"""CUDA-event timing of batched rectangle solves (warm L2): n, count list."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23180_b200 import configs, rectsolver
for spec in sys.argv[1:]:
    n, count = (int(x) for x in spec.split("x"))
    subs = configs.batch_rects(n, count, -100.0)
    plans = [rectsolver.plan_rect(s) for s in subs]
    rng = np.random.default_rng(0)
    f = [torch.as_tensor(rng.uniform(-1, 1, s.size), device="cuda") for s in subs]
    out = [torch.empty_like(x) for x in f]
    for _ in range(3):
        rectsolver.solve_rect_batched(plans, f, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 20
    e0.record()
    for _ in range(R):
        rectsolver.solve_rect_batched(plans, f, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    pts = sum(s.size for s in subs)
    print(f"{spec}: {ms * 1e3:.1f} us/apply, {pts / ms / 1e6:.2f} Gpts/s", flush=True)
