import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import fftddm_oracle as O
from paper_2509_23180_b200 import rectsolver
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from rects import make
for (m, n, half) in [(300, 4095, ("east",)), (300, 4095, ()), (64, 2047, ()), (2047, 2047, ())]:
    sub = make((m, n, 1.0 / n, 1.0 / n, 0.0, "DDDD", half))
    pl = rectsolver.plan_rect(sub)
    print(m, n, half, pl.info())
    f = np.random.default_rng(0).uniform(-1, 1, m * n)
    g = rectsolver.solve_rect(pl, f).values
    r = O.solve(O.plan(sub), f)
    E = O.apply_q_dd((g - r).reshape(m, n))   # error in spectral modes
    R = O.apply_q_dd(r.reshape(m, n))
    em = np.linalg.norm(E, axis=0) / np.linalg.norm(R, axis=0)
    bad = np.nonzero(em > 1e-10)[0]
    print("  rel err", np.linalg.norm(g - r) / np.linalg.norm(r), "bad modes", bad[:20], len(bad))
    er = np.linalg.norm((g - r).reshape(m, n), axis=1)
    print("  bad rows", np.nonzero(er > 1e-10 * np.linalg.norm(r) / np.sqrt(m))[0][:20])
