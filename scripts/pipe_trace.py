"""Dump the pipelined kernel's timeline at C2 (PR_PIPE_TRACE) and summarise it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PR_PIPE_TRACE"] = os.environ.get("PR_PIPE_TRACE", "gpurun_out/pipe_trace.txt")
from paper_2303_03848_b200 import parareal, synth  # noqa: E402
theta = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
net = synth.PINN_PAPER if "paper" in sys.argv else synth.PINN_3x20
p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0, fine_theta=theta)
with parareal.Context(p) as c:
    c.load_weights(synth.kaiming_net(net, seed=0))
    for _ in range(3):
        U, rep = c.solve()
    print(rep)
rows = [list(map(int, l.split())) for l in open(os.environ["PR_PIPE_TRACE"])]
t0 = min(r[2] for r in rows if r[2] > 0)
for k in range(4):
    ch = [(r[1], (r[2] - t0) / 1e3) for r in rows if r[0] == k and r[2] > 0]
    fs = [(r[1], (r[3] - t0) / 1e3, (r[4] - t0) / 1e3) for r in rows if r[0] == k and r[3] > 0]
    if ch:
        print("chain k=%d: first slice %d at %.1f us, last slice %d at %.1f us (%.2f us/slice)" % (
            k, ch[0][0], ch[0][1], ch[-1][0], ch[-1][1], (ch[-1][1] - ch[0][1]) / max(1, len(ch) - 1)))
    if fs:
        d = [e - s for _, s, e in fs]
        print("fine  k=%d: n=%d start %.1f end %.1f; n=%d start %.1f end %.1f; duration mean %.1f us" % (
            k, fs[0][0], fs[0][1], fs[0][2], fs[-1][0], fs[-1][1], fs[-1][2], sum(d) / len(d)))
print("k n chain_t fine_start fine_end")
for r in rows:
    if r[0] in (1, 2) and r[1] <= 6:
        print(r[0], r[1], *["%.1f" % ((v - t0) / 1e3) if v else "-" for v in r[2:]])
