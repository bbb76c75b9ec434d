"""Accuracy of the tensor-core PINN modes vs the fp64 oracle: one G application on a C5-like row
(M = 700, payoff x smooth modulation), max |gpu - ref| / max|ref| per (width, depth, mode)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2303_03848_b200 import parareal, synth
p = synth.portfolio(n_k=2, n_s=1, M=700, N=8)
U = oracle.payoff(p) * (1.0 + 0.05 * np.sin(np.arange(700) / 29.0))
for W, LH in [(64, 2), (64, 4), (64, 8), (128, 3), (128, 4), (128, 8), (256, 3), (256, 4), (256, 8)]:
    net = synth.kaiming_net([4] + [W] * LH + [1], seed=5 * W + LH)
    ref = oracle.pinn_G(p, net, 3, U)
    row = {"W": W, "LH": LH}
    for name, prec in (("fp16x3", 1), ("fp16x1", 4), ("bf16", 2)):
        with parareal.Context(p) as c:
            c.load_weights(net, precision=prec)
            got = c.apply_coarse(3, U.astype(np.float32))
        row[name] = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    print(json.dumps(row))
