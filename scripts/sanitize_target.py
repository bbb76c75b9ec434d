"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck), one kernel family each:
  python scripts/sanitize_target.py c1pipe|c2pipe|c2num|k2res|k2cn|k4|k4pp|c4
c1pipe/c2pipe: the pipelined cooperative kernel (PINN G); c2num: its numerical-G form; k2res: the
persistent bulk-copy/mbarrier K2 pass (>= 16 systems); k2cn: K2 tile kernels with CN; k4: the
tcgen05 PINN (split fp16); k4pp: the ping-pong TC kernel (bf16, resident weights); c4: K1 portfolio."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03848_b200 import parareal, synth  # noqa: E402

case = sys.argv[1]
net = None
prec = parareal.PREC_FP32
opt = {}
if case == "c1pipe":
    p = synth.config("C1", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
    net = synth.kaiming_net(synth.PINN_3x20, seed=0)
elif case == "c2pipe":
    p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0).replace(fine_steps=10)
    net = synth.kaiming_net(synth.PINN_3x20, seed=0)
elif case == "c2num":
    p = synth.config("C2", coarse=synth.COARSE_IMPLICIT_EULER, max_iter=3, tol=0.0).replace(fine_steps=10)
elif case == "k2res":
    p = synth.single(5000, 16, fine_steps=2, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=1, tol=0.0)
    opt[parareal.OPT_FINE_KERNEL] = 2
elif case == "k2cn":
    p = synth.single(5000, 4, fine_steps=2, fine_theta=0.5, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=1, tol=0.0)
    opt[parareal.OPT_FINE_KERNEL] = 2
elif case == "k4":
    p = synth.single(300, 4, fine_steps=4, coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
    net, prec = synth.kaiming_net([4, 64, 64, 64, 1], seed=1), parareal.PREC_FP16_TC
elif case == "k4pp":
    p = synth.single(600, 4, fine_steps=4, coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
    net, prec = synth.kaiming_net([4, 128, 128, 128, 1], seed=1), parareal.PREC_BF16_TC
elif case == "c4":
    p = synth.portfolio(n_k=4, n_s=4, M=256, N=16, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2, tol=0.0,
                        fine_steps=10)
elif case == "train":  # PINN trainer: k_train_grad (shared rows, stash) and k_adam (completion ticket)
    from paper_2303_03848_b200 import pinn_train
    mk = dict(K=1.0, sigma=0.2, r=0.05, T=1.0, L=4.0)
    with pinn_train.Trainer(synth.pinn2_net([2, 20, 20, 20, 1]), mk, synth.collocation(mk, 2000, 200, 200), batches=3) as tr:
        tr.epochs(2, 1e-2)
        print("train loss", tr.loss(), tr.batch_gradient(1)[0])
    raise SystemExit(0)
else:
    raise SystemExit("unknown case " + case)
with parareal.Context(p) as c:
    for k, v in opt.items():
        c.set_option(k, v)
    if net is not None:
        c.load_weights(net, precision=prec)
    U, rep = c.solve()
    print(case, "iterations", rep["iterations"], "launches", rep["kernel_launches"])
