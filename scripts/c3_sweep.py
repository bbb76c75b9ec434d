"""Times the C3 fine sweep (64 slices x 2^20 points x 100 IE steps, K2) as bench.py does:
ms_fine of a one-iteration graph-replayed solve, L2 flushed before each, median of 5."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_03848_b200 import parareal, synth
p = synth.config("C3", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with parareal.Context(p, stream=s.cuda_stream) as c:
    c.load_weights(synth.kaiming_net(synth.PINN_3x20, seed=0))
    c.set_option(parareal.OPT_USE_GRAPHS, 1)
    if os.environ.get("FINE_KERNEL"):
        c.set_option(parareal.OPT_FINE_KERNEL, int(os.environ["FINE_KERNEL"]))
    out = torch.empty((1, p.M), dtype=torch.float32, device="cuda")
    c.solve_device(out)
    ms = []
    for _ in range(5):
        flush.zero_(); torch.cuda.synchronize()
        ms.append(c.solve_device(out)["ms_fine"])
    t = statistics.median(ms)
    pts = float(p.M) * p.N * p.fine_steps
    print("C3 fine sweep %.3f ms  (%s)  %.1f G pt-steps/s  %.3f of HBM at 16 B, %.3f at 8 B" % (
        t, ["%.2f" % x for x in ms], pts / t / 1e6, 16 * pts / t / 1e6 / 6552.3, 8 * pts / t / 1e6 / 6552.3))
