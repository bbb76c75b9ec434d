"""ncu driver: the group-kernel PINN chain (paper's 10x50 net) at C2, blocking schedule."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
with parareal.Context(p) as c:
    c.load_weights(synth.kaiming_net(synth.PINN_PAPER, seed=0))
    c.set_option(parareal.OPT_PIPELINE, 1)
    U, rep = c.solve()
    print(rep)
