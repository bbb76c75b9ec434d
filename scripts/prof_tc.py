"""ncu target: the K4 chain at the C5 grid (k = 0 sweep), net 8x256 (or W LH from argv), precision from argv."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth
W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
LH = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prec = int(sys.argv[3]) if len(sys.argv) > 3 else parareal.PREC_FP16_TC
p = synth.config("C5", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
with parareal.Context(p) as c:
    c.load_weights(synth.kaiming_net([4] + [W] * LH + [1], seed=1), precision=prec)
    U, rep = c.solve()
    print(rep["ms_coarse"])
