"""ncu driver: the pipelined kernel with the paper's 10x50 net at C2 (K=3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
with parareal.Context(p) as c:
    c.load_weights(synth.kaiming_net(synth.PINN_PAPER, seed=0))
    for _ in range(2):
        U, rep = c.solve()
    print(rep)
