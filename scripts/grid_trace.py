"""Per-pass timeline of the grid-resident fine sweep (PR_GRID_TRACE) at the C3 grid."""
import os, sys
os.environ["PR_GRID_TRACE"] = "gpurun_out/grid_trace.txt"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_03848_b200 import parareal, synth
p = synth.single(1 << 20, 4, fine_steps=100, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=1, tol=0.0, T=4 * 100 / 6400.0)
U0 = synth.random_state(1, p.M, seed=3)
with parareal.Context(p) as c:
    c.set_option(parareal.OPT_FINE_KERNEL, 3)
    c.apply_fine(0, U0)
r = np.loadtxt(os.environ["PR_GRID_TRACE"], dtype=np.int64)
ps, cb, t0, t1, t2, t3, t4 = r.T
base = t0[t0 > 0].min()
npass = ps.max() + 1
for q in (10, 11, 50, 51):
    sel = ps == q
    print("pass", q, "start spread %.2f us" % ((t0[sel].max() - t0[sel].min()) / 1e3),
          "local+publish %.2f" % np.median((t1[sel] - t0[sel]) / 1e3),
          "lookback %.2f" % np.median((t2[sel] - t1[sel]) / 1e3),
          "barrier %.2f" % np.median((t3[sel] - t2[sel]) / 1e3),
          "rerun %.2f" % np.median((t4[sel] - t3[sel]) / 1e3),
          "max lookback %.2f" % ((t2[sel] - t1[sel]).max() / 1e3))
per = (t4[ps == npass - 1].max() - base) / npass / 1e3
print("mean per pass %.2f us over %d passes" % (per, npass))
