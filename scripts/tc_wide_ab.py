"""A/B of the one-tile K4 chain: 256 threads per 128-point tile (default) vs 128 (PR_TC_WIDE=0) at
the C5 grid (k = 0 sweep + k = 1 chain, ms_coarse min of 3), for the nets that run the one-tile
kernel: 8x256 in every mode (streamed weights), 4x128 / 8x128 split."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
for W, LH, prec, name in [(256, 8, parareal.PREC_FP16_TC, "split"), (256, 8, parareal.PREC_FP16X1_TC, "fp16x1"),
                          (256, 8, parareal.PREC_BF16_TC, "bf16"), (256, 4, parareal.PREC_FP16_TC, "split"),
                          (128, 4, parareal.PREC_FP16_TC, "split"), (128, 8, parareal.PREC_FP16_TC, "split"),
                          (64, 4, parareal.PREC_FP16_TC, "split"), (64, 6, parareal.PREC_FP16_TC, "split")]:
    p = synth.config("C5", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
    net = synth.kaiming_net([4] + [W] * LH + [1], seed=1)
    with parareal.Context(p) as c:
        c.load_weights(net, precision=prec)
        for _ in range(2):
            c.solve()
        ms = min(c.solve()[1]["ms_coarse"] for _ in range(3))
    evals = p.M * (p.N + p.N - 1)
    flop = evals * 2 * (4 * W + (LH - 1) * W * W + W)
    print(json.dumps(dict(W=W, LH=LH, mode=name, wide=os.environ.get("PR_TC_WIDE", "1"), ms_coarse=round(ms, 3),
                          model_tflops=round(flop / ms / 1e9, 1))), flush=True)
