"""K3 throughput mode at C3 (2^20 points x 64 slices, 3x20 net): coarse-chain time per kernel path
(PR_OPT_PINN_KERNEL 0 auto = constant-bank weights, 1 = shared-memory weights, PTS points/thread)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = synth.config(cfg, coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
for opt in (0, 1):
    with parareal.Context(p) as c:
        c.load_weights(synth.kaiming_net(synth.PINN_3x20, seed=0))
        c.set_option(parareal.OPT_PINN_KERNEL, opt)
        out = torch.empty((p.B, p.M), dtype=torch.float32, device="cuda")
        c.solve_device(out)
        ms = [c.solve_device(out)["ms_coarse"] for _ in range(3)]
        t = statistics.median(ms) / 2  # k = 0 chain over N slices + k = 1 chain over N-1 slices
        evals = p.B * p.M * p.N
        print("%s opt=%d coarse chain %.3f ms  %.2f G evals/s" % (cfg, opt, t, evals / t / 1e6), flush=True)
