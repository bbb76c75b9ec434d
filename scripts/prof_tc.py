"""ncu target: one K4 coarse launch at the C5 grid (2^18 points), W x LH net, precision arg."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
W, LH, prec = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = synth.config("C5", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
with parareal.Context(p) as c:
    c.load_weights(synth.kaiming_net([4] + [W] * LH + [1], seed=1), precision=prec)
    U = synth.random_state(1, p.M, seed=1)
    c.apply_coarse(3, U)
