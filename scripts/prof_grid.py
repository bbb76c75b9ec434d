"""One C3-grid fine sweep on the grid-resident kernel (ncu target): 2^20 points, 4 slices x 100 steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_03848_b200 import parareal, synth
p = synth.single(1 << 20, 4, fine_steps=100, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=1, tol=0.0, T=4 * 100 / 6400.0)
U0 = synth.random_state(1, p.M, seed=3)
with parareal.Context(p) as c:
    c.set_option(parareal.OPT_FINE_KERNEL, int(os.environ.get("FINE_KERNEL", "3")))
    out = c.apply_fine(0, U0)
    print("ok", float(np.abs(out).max()))
