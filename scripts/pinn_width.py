"""PINN-width sweep at the C5 grid (2^18 points x 64 slices): coarse-chain point-evals/s per
(width, depth, precision).  One Parareal iteration (k=0 sweep + k=1 chain) per solve."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
res = []
for W, LH, prec in [(20, 3, 0), (64, 4, 0), (64, 4, 1), (64, 8, 1), (128, 4, 1), (256, 4, 1), (256, 8, 1), (256, 8, 2),
                    (64, 4, 4), (64, 8, 4), (128, 4, 4), (256, 4, 4), (256, 8, 4)]:
    p = synth.config("C5", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
    net = synth.kaiming_net([4] + [W] * LH + [1], seed=1)
    with parareal.Context(p) as c:
        c.load_weights(net, precision=prec)
        for _ in range(2):
            _, rep = c.solve()
        ms = min(c.solve()[1]["ms_coarse"] for _ in range(3))
    evals = p.M * (p.N + p.N - 1)
    flop = evals * 2 * (4 * W + (LH - 1) * W * W + W)
    r = dict(W=W, LH=LH, prec={0: "fp32", 1: "fp16x3_tc", 2: "bf16_tc", 4: "fp16x1_tc"}[prec], ms_coarse=ms, evals_per_s=evals / ms * 1e3,
             model_tflops=flop / ms / 1e9)
    print(json.dumps(r)); res.append(r)
json.dump(res, open("gpurun_out/pinn_width.json", "w"), indent=1)
