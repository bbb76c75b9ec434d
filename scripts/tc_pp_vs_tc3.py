"""A/B: nets where the ping-pong K4 kernel is chosen (split mode) vs the layer-pipelined tc3
(run with PR_TC_PINGPONG=0 PR_TC_PIPE=3), C5 grid, ms_coarse of k = 0 + k = 1 (min of 3)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
for W, LH in [(128, 3), (64, 8), (128, 2), (256, 2)]:
    p = synth.config("C5", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
    with parareal.Context(p) as c:
        c.load_weights(synth.kaiming_net([4] + [W] * LH + [1], seed=1), precision=parareal.PREC_FP16_TC)
        for _ in range(2):
            c.solve()
        ms = min(c.solve()[1]["ms_coarse"] for _ in range(3))
    print(json.dumps(dict(W=W, LH=LH, pingpong=os.environ.get("PR_TC_PINGPONG", "1"), pipe=os.environ.get("PR_TC_PIPE", "1"),
                          ms_coarse=round(ms, 3))), flush=True)
