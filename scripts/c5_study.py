"""C5 study (the NEXT-3 follow-on): iterations-to-tolerance vs coarse cost
at 2^18 grid points × 64 slices × 100 implicit-Euler fine steps per slice, one B200.

PINN coarse propagators are trained on the GPU (pinn_train, the paper's schedule: P:190
collocation counts, P:210-211 5000 epochs at 1e-2 + 800 at 1e-3, 10 shuffled batches per epoch)
for 2-input tanh nets W ∈ {20, 64} × L_h ∈ {4, 6, 8} (the trainer's widths; W = 256 is not
trainable here), then each runs Parareal as G:
  * δ^1 … δ^16 of a fixed-K solve → K(tol) = the first k with δ^k < tol (the library's stop rule,
    evaluated on the same history) for tol ∈ {1e-4, 1e-5, 1e-6, 1e-7};
  * per-iteration coarse and fine time (ms_coarse / K, ms_fine / K of the blocking schedule);
  * a converged solve at tol = 1e-6 (max_iter 32): iterations, time, and its distance from the
    GPU serial fine solution;
W = 64 nets also with the split-fp16 tensor-core chain (K4).  Numerical G (IE, n_c = 1 and 50
steps per slice) for comparison.  Writes profiles/r02/c5_study.{json,md}.
No oracle is used (measurement script): the closed form for Ṽ(0, S) is evaluated inline."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_03848_b200 import parareal, pinn_train, synth

MK = dict(K=1.0, sigma=0.2, r=0.05, T=1.0, L=4.0)
TOLS = (1e-4, 1e-5, 1e-6, 1e-7)
KFIX = 16
OUT = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c5_study"
os.makedirs(OUT, exist_ok=True)


def bs_call(S, K, r, s, T):
    if S <= 0:
        return 0.0
    d1 = (math.log(S / K) + (r + 0.5 * s * s) * T) / (s * math.sqrt(T))
    d2 = d1 - s * math.sqrt(T)
    Phi = lambda x: 0.5 * (1.0 + math.erf(x / math.sqrt(2.0)))
    return S * Phi(d1) - K * math.exp(-r * T) * Phi(d2)


def k_of(delta, tol):
    for k, d in enumerate(delta, 1):
        if d < tol:
            return k
    return None


def study(p0, net=None, prec=parareal.PREC_FP32, coarse_steps=None, kfix=KFIX, converge=True):
    row = {}
    kw = dict(max_iter=kfix, tol=0.0)
    if coarse_steps:
        kw.update(coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=coarse_steps)
    p = p0.replace(**kw)
    with parareal.Context(p) as c:
        if net is not None:
            c.load_weights(net, precision=prec)
            S = np.arange(1, p.M + 1) * MK["L"] / (p.M + 1)
            G0 = c.apply_coarse(p.N - 1, np.zeros((1, p.M), np.float32))[0]  # 2-input G: Ṽ(t = 0, S)
            sub = slice(None, None, 64)
            ref = np.array([bs_call(s, MK["K"], MK["r"], MK["sigma"], MK["T"]) for s in S[sub]])
            row["G_t0_vs_closed_form"] = float(np.linalg.norm(G0[sub] - ref) / np.linalg.norm(ref))
        c.solve()  # warm-up
        U, rep = c.solve()
        d = [float(x) for x in rep["delta"]]
        row["delta"] = d
        row["K_of_tol"] = {"%g" % t: k_of(d, t) for t in TOLS}
        row["coarse_ms_per_iter"] = rep["ms_coarse"] / (kfix + 1)  # k = 0 sweep + K chains
        row["fine_ms_per_iter"] = rep["ms_fine"] / kfix
        row["fixedK_ms_total"] = rep["ms_total"]
        fine, ms_sf = c.serial_fine()
        row["serial_fine_ms"] = ms_sf
    if not converge:
        return row
    pc = p.replace(max_iter=32, tol=1e-6)
    with parareal.Context(pc) as c:
        if net is not None:
            c.load_weights(net, precision=prec)
        c.solve()
        U, rep = c.solve()
        row["tol1e-6"] = {"iterations": int(rep["iterations"]), "converged": bool(rep["converged"]),
                          "ms_total": rep["ms_total"],
                          "speedup_vs_serial_fine": row["serial_fine_ms"] / rep["ms_total"],
                          "rel_to_serial_fine": float(np.max(np.abs(U - fine)) / np.max(np.abs(fine)))}
    return row


p0 = synth.config("C5", coarse=synth.COARSE_PINN)
rows = []
for W in (20, 64):
    for LH in (4, 6, 8):
        dims = [2] + [W] * LH + [1]
        sets = synth.collocation(MK, *synth.PAPER_COLLOCATION, seed=0)
        t0 = time.perf_counter()
        try:
            tr = pinn_train.Trainer(synth.pinn2_net(dims, seed=0), MK, sets, batches=10, seed=0)
        except parareal.PararealError as e:  # the trainer's shared-memory budget (8 x 64)
            rows.append({"net": "%dx%d" % (LH, W), "precision": "—", "untrainable": str(e)})
            print("skip %dx%d: %s" % (LH, W, e), flush=True)
            continue
        with tr:
            l0 = tr.loss()
            tr.epochs(5000, 1e-2, history=False)
            tr.epochs(800, 1e-3, history=False)
            l1 = tr.loss()
            net = tr.net()
        t_train = time.perf_counter() - t0
        for prec, pname in ((parareal.PREC_FP32, "fp32"),) + (((parareal.PREC_FP16_TC, "split-fp16 TC"),) if W == 64 else ()):
            r = study(p0, net, prec)
            r.update(net="%dx%d" % (LH, W), precision=pname, train_s=t_train, loss_initial=float(np.sum(l0)),
                     loss_final=float(np.sum(l1)))
            rows.append(r)
            print(json.dumps({k: v for k, v in r.items() if k != "delta"}), flush=True)
# W = 256 (not trainable here): the coarse cost of random 4-input nets on the split-fp16 TC chain
# (iterations-to-tolerance from random weights is N by construction)
for LH in (4, 8):
    net = synth.kaiming_net([4] + [256] * LH + [1], seed=0)
    r = study(p0, net, parareal.PREC_FP16_TC, kfix=2, converge=False)
    r.update(net="%dx256 (random, 4-input)" % LH, precision="split-fp16 TC")
    rows.append(r)
    print(json.dumps({k: v for k, v in r.items() if k != "delta"}), flush=True)
for nc in (1, 50):
    r = study(p0, coarse_steps=nc)
    r.update(net="IE n_c=%d" % nc, precision="fp64")
    rows.append(r)
    print(json.dumps({k: v for k, v in r.items() if k != "delta"}), flush=True)
json.dump({"workload": "C5: 2^18 points x 64 slices x 100 IE steps/slice, European call K=1 r=0.05 sigma=0.2 T=1 L=4",
           "rows": rows}, open(os.path.join(OUT, "c5_study.json"), "w"), indent=1)
lines = ["| G | precision | train s | final loss | ‖Ṽ(0)−BS‖/‖BS‖ | δ¹ | K(1e-5) | K(1e-6) | K(1e-7) | coarse ms/iter | fine ms/iter | tol 1e-6: K, ms | serial fine ms | speedup |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    if "untrainable" in r:
        lines.append("| %s | — | %s |" % (r["net"], r["untrainable"]) + " |" * 11)
        continue
    if "tol1e-6" not in r:
        lines.append("| %s | %s | — | — | — | %.2e | — | — | — | %.3f | %.3f | — | %.1f | — |" % (
            r["net"], r["precision"], r["delta"][0], r["coarse_ms_per_iter"], r["fine_ms_per_iter"], r["serial_fine_ms"]))
        continue
    t = r["tol1e-6"]
    lines.append("| %s | %s | %s | %s | %s | %.2e | %s | %s | %s | %.3f | %.3f | %d%s, %.1f | %.1f | %.2f× |" % (
        r["net"], r["precision"], "%.1f" % r["train_s"] if "train_s" in r else "—",
        "%.2e" % r["loss_final"] if "loss_final" in r else "—",
        "%.2e" % r["G_t0_vs_closed_form"] if "G_t0_vs_closed_form" in r else "—", r["delta"][0],
        r["K_of_tol"]["1e-05"] or ">16", r["K_of_tol"]["1e-06"] or ">16", r["K_of_tol"]["1e-07"] or ">16", r["coarse_ms_per_iter"],
        r["fine_ms_per_iter"], t["iterations"], "" if t["converged"] else " (not conv.)", t["ms_total"],
        r["serial_fine_ms"], t["speedup_vs_serial_fine"]))
open(os.path.join(OUT, "c5_study.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
