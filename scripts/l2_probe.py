"""Probe: K2 fine-sweep time per point-step vs working-set size (does an L2-resident slice group
run faster than the HBM-streamed full sweep?).  python scripts/l2_probe.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2303_03848_b200 import parareal, synth  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for M, N in [(1 << 20, 64)] if os.environ.get("PR_PROBE_ONE") else [(1 << 20, 64), (1 << 20, 16), (1 << 19, 16), (1 << 18, 32), (1 << 18, 16), (1 << 17, 32)]:
    p = synth.single(M, N, coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
    with parareal.Context(p) as ctx:
        ctx.load_weights(synth.kaiming_net(synth.PINN_3x20, seed=0))
        ctx.set_option(parareal.OPT_USE_GRAPHS, 1)
        out = torch.empty((p.B, p.M), dtype=torch.float32, device="cuda")
        ctx.solve_device(out)
        ms = []
        for _ in range(5):
            flush.zero_()
            torch.cuda.synchronize()
            ms.append(ctx.solve_device(out)["ms_fine"])
        t = statistics.median(ms)
        ws = 2 * M * N * 4 / 2**20
        print(f"M={M} N={N} state(X+Y)={ws:.0f} MiB  ms_fine={t:.3f}  ns/pt-step={t*1e6/(M*N*100):.4f}  "
              f"GB/s@16B={16*M*N*100/t/1e6:.0f}", flush=True)
