"""ncu target: the blocking C2 schedule (PR_OPT_PIPELINE = 1), whose coarse chain is the
latency-mode k_pinn_chain_split over 32 slices (the pipelined chain's evaluator)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth
p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
with parareal.Context(p) as c:
    c.load_weights(synth.kaiming_net(synth.PINN_3x20, seed=0))
    c.set_option(parareal.OPT_PIPELINE, 1)
    U, rep = c.solve()
    print(rep)
