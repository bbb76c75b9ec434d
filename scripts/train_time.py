"""Times the paper's training schedule (P:190 sets, P:210-211 epochs) on the GPU trainer."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_03848_b200 import pinn_train, synth
MK = dict(K=1.0, sigma=0.2, r=0.05, T=1.0, L=4.0)
dims = [2] + [int(w) for w in (sys.argv[1] if len(sys.argv) > 1 else "20,20,20").split(",")] + [1]
sets = synth.collocation(MK, *synth.PAPER_COLLOCATION, seed=0)
with pinn_train.Trainer(synth.pinn2_net(dims, seed=0), MK, sets, batches=10, seed=0) as tr:
    tr.epochs(20, 1e-2, history=False)  # warm-up
    t0 = time.perf_counter(); tr.epochs(5000, 1e-2, history=False); t1 = time.perf_counter()
    h = tr.epochs(800, 1e-3); t2 = time.perf_counter()
    print(dims, "5000 epochs %.3f s, 800 epochs %.3f s, %.2f us/step, final full loss %s" % (
        t1 - t0, t2 - t1, 1e6 * (t2 - t0) / (5800 * 10), tr.loss()))
