"""Partition debugging: 5 x 1023^2 batch against the oracle, per subdomain, with the row
ranges around every subdomain start (FD_PHASE_TIMING_ALL output parsed from stderr by the caller)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import fftddm_oracle as O
from paper_2509_23180_b200 import configs, rectsolver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1023
subs = configs.batch_rects(n, 5, -10.0)
r = np.random.default_rng(0)
f = [r.uniform(-1, 1, s.size) for s in subs]
plans = [rectsolver.plan_rect(s) for s in subs]
outs = rectsolver.solve_rect_batched(plans, f)
bad = []
for sid, (s, fi, o) in enumerate(zip(subs, f, outs)):
    ref = O.solve(O.plan(s), fi)
    v = o.cpu().numpy()
    e = np.linalg.norm(v - ref) / np.linalg.norm(ref)
    if not e < 1e-11:
        bad.append((sid, float(e)))
print("BAD", bad)
