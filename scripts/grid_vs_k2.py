"""Fine sweep time of the grid-resident kernel (3) vs K2 (2) over nsl slices of 2^20 points x 100
IE steps (one Parareal iteration's fine sweep; ms_fine of a graph-replayed solve, min of 3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth
for nsl in (1, 2, 4, 8, 16):
    p = synth.single(1 << 20, nsl, fine_steps=100, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=1, tol=0.0,
                     T=nsl * 100 / 6400.0)
    row = {}
    for fk in (2, 3):
        with parareal.Context(p) as c:
            c.set_option(parareal.OPT_FINE_KERNEL, fk)
            for _ in range(2):
                c.solve()
            row[fk] = min(c.solve()[1]["ms_fine"] for _ in range(3))
    print("nsl %2d  K2 %.3f ms  grid %.3f ms  ratio %.2f" % (nsl, row[2], row[3], row[2] / row[3]))
