"""K2R grid-resident fine sweep vs the oracle and vs K2 on small and C3-size problems."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2303_03848_b200 import parareal, synth
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_helpers import assert_close, rel_err
for M, N, nf in [(3000, 4, 10), (5000, 5, 7), (70000, 4, 5), (1 << 18, 4, 6)]:
    p = synth.single(M, N, fine_steps=nf, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2, tol=0.0)
    U0 = synth.random_state(1, M, seed=3)
    res = {}
    for fk in (2, 3):
        with parareal.Context(p) as c:
            c.set_option(parareal.OPT_FINE_KERNEL, fk)
            res[fk] = c.apply_fine(1, U0)
    ref = oracle.fine(p, 1, U0.astype(np.float64))
    print(M, N, nf, "grid vs oracle", rel_err(res[3], ref), "K2 vs oracle", rel_err(res[2], ref))
    with parareal.Context(p) as c:
        c.set_option(parareal.OPT_FINE_KERNEL, 3)
        U, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    refU, refd, K, _ = oracle.parareal(p)
    print("  parareal grid vs oracle", rel_err(it, refU), rep["iterations"], K)
