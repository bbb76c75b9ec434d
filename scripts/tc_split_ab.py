"""A/B of the split-fp16 K4 chain: ping-pong (default) vs one-tile (PR_TC_PINGPONG=2) at the C5 grid."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
for W, LH in [(64, 8), (128, 3), (128, 4), (128, 8)]:
    p = synth.config("C5", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
    net = synth.kaiming_net([4] + [W] * LH + [1], seed=1)
    with parareal.Context(p) as c:
        c.load_weights(net, precision=parareal.PREC_FP16_TC)
        for _ in range(2):
            c.solve()
        ms = min(c.solve()[1]["ms_coarse"] for _ in range(3))
    evals = p.M * (p.N + p.N - 1)
    flop = evals * 2 * (4 * W + (LH - 1) * W * W + W)
    print(json.dumps(dict(W=W, LH=LH, pingpong=os.environ.get("PR_TC_PINGPONG", "1"), ms_coarse=ms,
                          evals_per_s=evals / ms * 1e3, model_tflops=flop / ms / 1e9)))
