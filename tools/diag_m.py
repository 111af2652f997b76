"""Rectangle solve vs oracle over several m for given n (localises kernel bugs)."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import fftddm_oracle as O
from paper_2509_23180_b200 import rectsolver
from rects import make
n = int(sys.argv[1])
for m in [int(x) for x in sys.argv[2].split(",")]:
    sub = make((m, n, 1.0 / n, 1.0 / n, 0.0, "DDDD", ()))
    pl = rectsolver.plan_rect(sub)
    f = np.random.default_rng(0).uniform(-1, 1, m * n)
    g = rectsolver.solve_rect(pl, f).values
    r = O.solve(O.plan(sub), f)
    E = O.apply_q_dd((g - r).reshape(m, n)); R = O.apply_q_dd(r.reshape(m, n))
    em = np.linalg.norm(E, axis=0) / np.linalg.norm(R, axis=0)
    er = np.linalg.norm((g - r).reshape(m, n), axis=1) / (np.linalg.norm(r) / np.sqrt(m))
    bad = np.nonzero(em > 1e-10)[0]; badr = np.nonzero(er > 1e-10)[0]
    print(f"m={m} rel {np.linalg.norm(g - r) / np.linalg.norm(r):.2e} bad modes {len(bad)} {bad[:8]} bad rows {len(badr)} {badr[:8]}", flush=True)
