"""Blocking C2 schedule (PR_OPT_PIPELINE = 1): coarse-chain phase time (k = 0 sweep + K chains of the
latency-mode k_pinn_chain_split), min of 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth
p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
with parareal.Context(p) as c:
    c.load_weights(synth.kaiming_net(synth.PINN_3x20, seed=0))
    c.set_option(parareal.OPT_PIPELINE, 1)
    for _ in range(3):
        c.solve()
    print("blocking C2 ms_coarse %.4f" % min(c.solve()[1]["ms_coarse"] for _ in range(5)))
