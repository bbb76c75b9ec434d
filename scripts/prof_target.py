"""Small drivers for ncu captures (one workload each): python scripts/prof_target.py c3|c4|c2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = {"c2": "C2", "c3": "C3", "c4": "C4"}[which]
coarse = synth.COARSE_IMPLICIT_EULER if "ie" in sys.argv else synth.COARSE_PINN
p = synth.config(cfg, coarse=coarse, max_iter=int(os.environ.get("PR_ITERS", "1")), tol=0.0)
with parareal.Context(p) as c:
    if coarse == synth.COARSE_PINN:
        c.load_weights(synth.kaiming_net(synth.PINN_3x20, seed=0))
    for _ in range(int(os.environ.get("PR_REPS", "1"))):
        U, rep = c.solve()
    print(which, rep)
