"""One fine sweep on the grid-resident kernel K2R (ncu target): 2^20 points x NSL slices x 100 IE
steps (NSL from argv, default 4; 64 = the C3 sweep, one launch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_03848_b200 import parareal, synth
nsl = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = synth.single(1 << 20, nsl, fine_steps=100, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=1, tol=0.0,
                 T=nsl * 100 / 6400.0)
with parareal.Context(p) as c:
    c.set_option(parareal.OPT_FINE_KERNEL, int(os.environ.get("FINE_KERNEL", "3")))
    U, rep = c.solve()
    print("ok", rep["ms_fine"], float(np.abs(U).max()))
