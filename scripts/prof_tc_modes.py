"""One K4 chain launch per tensor-core mode at the C5 grid (8x256 net) for ncu: split fp16,
single-pass fp16, bf16 (python scripts/prof_tc_modes.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
p = synth.config("C5", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
net = synth.kaiming_net([4] + [256] * 8 + [1], seed=1)
for prec in (parareal.PREC_FP16_TC, parareal.PREC_FP16X1_TC, parareal.PREC_BF16_TC):
    with parareal.Context(p) as c:
        c.load_weights(net, precision=prec)
        _, rep = c.solve()
        print(prec, rep["ms_coarse"])
