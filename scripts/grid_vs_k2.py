"""Fine sweep time of the grid-resident kernel (3) vs K2 (2) over nsl slices of M points x 100
IE steps (one Parareal iteration's fine sweep; ms_fine of a graph-replayed solve, min of 3).
Usage: grid_vs_k2.py [M ...]  (default 2^20)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth
Ms = [int(eval(a)) for a in sys.argv[1:]] or [1 << 20]
for M in Ms:
    for nsl in ((1, 3, 4, 8, 16, 64) if len(Ms) == 1 else (4, 16, 64)):
        p = synth.single(M, nsl, fine_steps=100, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=1, tol=0.0,
                         T=nsl * 100 / 6400.0)
        row = {}
        for fk in (2, 3):
            with parareal.Context(p) as c:
                c.set_option(parareal.OPT_FINE_KERNEL, fk)
                for _ in range(2):
                    c.solve()
                row[fk] = min(c.solve()[1]["ms_fine"] for _ in range(3))
        print("M %7d nsl %2d  K2 %.3f ms  grid %.3f ms  ratio %.2f" % (M, nsl, row[2], row[3], row[2] / row[3]))
