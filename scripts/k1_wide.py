"""Serial fine solve time at C2 (k_resident_chain: 128 threads x 8 points vs PR_K1_WIDE=1: 256 x 4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth
p = synth.config("C2", coarse=synth.COARSE_IMPLICIT_EULER, max_iter=1, tol=0.0)
with parareal.Context(p) as c:
    for _ in range(3):
        c.serial_fine()
    print("PR_K1_WIDE=%s serial fine %.3f ms" % (os.environ.get("PR_K1_WIDE", "0"), min(c.serial_fine()[1] for _ in range(5))))
