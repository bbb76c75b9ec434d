#!/usr/bin/env python
"""Benchmark of the Parareal + PINN hot path (BASELINE.json metric) on N GPUs.

One step = one full Parareal solve (all SURVEY.md §8(a) rows: payoff, k=0 coarse sweep,
K fine sweeps with the correction + coarse chain, δ reductions, output) through the C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--coarse pinn|ie] [--iters 3]
  python bench.py --impl reference ...   # the CPU oracle as the reference arm (rank 0 only)

Default workload: configs[1] (C2: 1024 points x 32 slices, PINN 3x20 coarse, fixed K=3 as the
paper reports runtimes for K=3).  value = grid-point-steps of the problem solved
(B·M·N·n_f per solve: the serial fine work Parareal replaces) per second of device time.
Inputs (C2) are far below L2 size, so L2 is flushed (256 MiB write) before every timed step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Parareal speedup vs serial fine; fine grid-point-steps/s; PINN evals/s"
UNIT = "grid-point-steps/s"
FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--coarse", default="pinn", choices=["pinn", "ie"])
    ap.add_argument("--iters", type=int, default=3, help="fixed Parareal iterations K (tol = 0)")
    ap.add_argument("--coarse-steps", type=int, default=1,
                    help="implicit-Euler steps per slice of the numerical coarse G (--coarse ie; paper ratio n_f/2 = 50)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3-sweep", action="store_true", help="skip the C3 fine-sweep HBM roofline leg")
    ap.add_argument("--no-training", action="store_true", help="skip the PINN-training leg (NEXT-3)")
    ap.add_argument("--no-graphs", action="store_true", help="eager launches instead of the captured CUDA graph")
    ap.add_argument("--pinn-width", type=int, default=20, help="PINN hidden width (C5 sweep: 20/64/256)")
    ap.add_argument("--pinn-layers", type=int, default=3, help="PINN hidden layers")
    ap.add_argument("--pinn-prec", default="fp32", choices=["fp32", "fp16tc", "bf16tc"],
                    help="PINN arithmetic: fp32 SIMT, split-fp16 tensor cores (fp32-level accuracy), bf16 tensor cores")
    ap.add_argument("--fine-theta", type=float, default=1.0,
                    help="fine theta-step: 1 implicit Euler (default, reading Q1), 0.5 Crank-Nicolson (NEXT-1)")
    return ap.parse_args()


def problem_for(args):
    from paper_2303_03848_b200 import synth
    coarse = synth.COARSE_PINN if args.coarse == "pinn" else synth.COARSE_IMPLICIT_EULER
    p = synth.config(args.config, coarse=coarse, coarse_steps=args.coarse_steps, tol=0.0, fine_theta=args.fine_theta)
    return p.replace(max_iter=min(args.iters, p.N))


def work_units(p) -> float:
    """Grid-point-steps of the problem: B·M·N·n_f (the serial fine solve's point-steps)."""
    return float(p.B) * p.M * p.N * p.fine_steps


PREC_CODE = {"fp32": 0, "fp16tc": 1, "bf16tc": 2}


def pinn_dims(args):
    return [4] + [args.pinn_width] * args.pinn_layers + [1]


def pinn_flops(dims) -> float:
    return float(sum(2 * dims[l] * dims[l + 1] for l in range(len(dims) - 1)))


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # let nvidia-smi initialise (and take a first sample) before the timed region
            while not self.rows and time.time() - t0 < 2.0:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


ALU = None


def alu_peaks():
    """fp64 / fp32 FMA peaks measured on this pool's B200 by scripts/peaks_microbench.cu
    (profiles/r02/peaks.json); the nominal unit-count figure only if that file is missing."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "peaks.json")) as f:
            d = json.load(f)
        return {"fp64": float(d["fp64_fma_tflops"]), "fp32": float(d["fp32_fma_tflops"]),
                "src": "measured (scripts/peaks_microbench.cu, profiles/r02/peaks.json)"}
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# --------------------------------------------------------------------------- reference arm
def cpu_oracle_run(p, net, budget_s: float, max_runs: int, threads: int = 1):
    """Time the CPU oracle (as it stands) on the full workload; returns (sec per solve, runs, cores).
    threads > 1: its threaded-fine variant (fine sweep slices on std::threads, bitwise the same)."""
    import oracle
    times = []
    t_start = time.perf_counter()
    while len(times) < max_runs:
        t0 = time.perf_counter()
        oracle.parareal(p, net, threads=threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    return statistics.mean(times), len(times), threads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2303_03848_b200 import synth
    p = problem_for(args)
    net = synth.kaiming_net(pinn_dims(args), seed=0) if p.coarse == synth.COARSE_PINN else None
    import oracle  # (the oracle evaluates the net in fp64 whatever --pinn-prec says)
    for _ in range(max(0, min(args.warmup, 1))):
        oracle.parareal(p, net)
    per, runs, cores = cpu_oracle_run(p, net, budget_s=1e9, max_runs=max(1, args.steps))
    value = work_units(p) / per
    sample = "full %s workload (M=%d, N=%d, B=%d, K=%d), %d timed solves" % (args.config, p.M, p.N, p.B,
                                                                             p.max_iter, runs)
    line = {"impl": "reference", "cpu_model": cpu_model(), "host_threads": os.cpu_count(), "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": runs, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, p),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def step_stats(ms):
    """Per-step device times: median, mean ± std (the paper reports mean ± std over 5 runs)."""
    return {"n": len(ms), "median": statistics.median(ms), "mean": statistics.mean(ms),
            "std": statistics.stdev(ms) if len(ms) > 1 else 0.0, "min": min(ms), "max": max(ms)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def config_dict(args, p):
    return {"workload": "%s: European call, M=%d grid points x N=%d slices x B=%d instances, %d %s fine "
                        "steps/slice, %s coarse, K=%d fixed iterations" % (
                            args.config, p.M, p.N, p.B, p.fine_steps,
                            "IE" if p.fine_theta == 1.0 else ("CN" if p.fine_theta == 0.5 else "theta=%g" % p.fine_theta),
                            ("PINN %s tanh (%s)" % (pinn_dims(args), args.pinn_prec)) if args.coarse == "pinn"
                            else "implicit-Euler (%d step%s/slice)" % (p.coarse_steps, "" if p.coarse_steps == 1 else "s"),
                            p.max_iter),
            "M": p.M, "N": p.N, "B": p.B, "fine_steps": p.fine_steps, "fine_theta": p.fine_theta, "K": p.max_iter,
            "coarse": args.coarse, "parallelism": "time-slices/%d" % args.gpus,
            "cuda_graph": (not args.no_graphs) and args.gpus == 1,
            "timed_replay": "lean stream-ordered graph replay (PR_OPT_USE_GRAPHS=2)" if not args.no_graphs else "eager",
            "l2": "flushed (256 MiB write) before every timed step" if p.M * p.B * 4 * (p.N + 1) * 3 < (126 << 20)
            else "working set larger than L2"}


def ncu_traffic(kernel_prefix):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of a kernel, from the committed
    `ncu --set full` capture summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
    except Exception:
        return None
    for name, rec in d.get("kernels", {}).items():
        if name.startswith(kernel_prefix):
            return rec
    return None


def roofline(p, ph, K, world, rank, pk, pk_src, clk_mhz, n_sm, synth, dims=None, tc_prec=None):
    """Roofline of the step's dominant kernel (DESIGN.md §6 work per unit)."""
    nloc = p.N // world
    if ph["ms_fine"] >= ph["ms_coarse"]:
        # average active slices per fine sweep on this rank (slices n >= k-1 at iteration k)
        act = sum(max(0, nloc - max(0, k - 1 - rank * nloc)) for k in range(1, K + 1)) / K
        pt_steps = float(p.B) * p.M * p.fine_steps * act
        sweep_s = ph["ms_fine"] / K / 1e3
        if p.M <= 2048:
            piped = ph["ms_fine"] == ph["ms_coarse"]  # the pipelined schedule reports its overlapped time in both
            pipe_name = ("k_parareal_pipe_num (pipelined schedule, numerical G; fine role = K1, fp64)"
                         if p.coarse == synth.COARSE_IMPLICIT_EULER
                         else "k_parareal_pipe (pipelined schedule; fine role = K1, fp64)")
            roof = {"kernel": pipe_name if piped
                    else "k_fine_sweep (resident K1, fp64)", "bound": "alu",
                    "note": "latency-bound at this size: each implicit step is two dependent scans over "
                            "one system per CTA (0.5 us/step), one CTA per slice on 148 SMs; the fraction "
                            "of the fp64 pipe is small by construction (DESIGN.md 6, 11)",
                    "achieved": 9.0 * pt_steps / sweep_s / 1e12,
                    "peak": ALU["fp64"] if ALU else n_sm * 64 * 2 * clk_mhz * 1e6 / 1e12,
                    "unit": "TFLOP/s", "peak_source": ALU["src"] if ALU else
                    "fp64 pipe: %d SMs x 64 FMA/clk x 2 x %.0f MHz (nominal)" % (n_sm, clk_mhz),
                    "work_per_unit": "9 fp64 flop per point-step", "launch_unit": "one sweep"}
            tr = ncu_traffic("k_parareal_pipe" if piped else "k_fine_sweep")
        else:
            grid = p.fine_theta == 1.0 and p.B == 1
            kname = ("k_fine_grid / k_pass_res2 (K2R grid-resident solver where its cost model wins, else K2)"
                     if grid else "k_streamed_pass (K2, Crank-Nicolson tile pass)")
            roof = {"kernel": kname, "bound": "hbm",
                    "achieved": 8.0 * pt_steps / sweep_s / 1e9,
                    "peak": float(pk["hbm_gbs"]), "unit": "GB/s", "peak_source": pk_src,
                    "work_per_unit": "8 B per point-step (SURVEY 8(d) algorithmic: one fp32 read + write; "
                                     "the two-pass kernel moves 16)", "launch_unit": "one sweep"}
            tr = ncu_traffic("k_fine_grid" if grid else "k_streamed_pass")
    else:
        evals = float(p.B) * p.M * nloc
        chain_s = ph["ms_coarse"] / (K + 1) / 1e3
        if p.coarse == synth.COARSE_PINN and tc_prec:
            fl = pinn_flops(dims)
            w = dims[1] if dims else 0
            kname = ("k_pinn_chain_tc3" if tc_prec == "fp16tc" and w == 256 else "k_pinn_chain_tc")
            roof = {"kernel": "%s (K4, tcgen05 %s)" % (kname, tc_prec), "bound": "tensor",
                    "achieved": fl * evals / chain_s / 1e12,
                    "peak": float(pk["bf16_tflops"]), "unit": "TFLOP/s",
                    "peak_source": "measured dense bf16 (fp16 runs at the bf16 rate)",
                    "work_per_unit": "%.0f algorithmic flop per point-eval (the split-fp16 mode issues 3x)" % fl,
                    "launch_unit": "one coarse chain"}
            tr = ncu_traffic(kname + ("<" if kname == "k_pinn_chain_tc" else ""))
        elif p.coarse == synth.COARSE_PINN:
            fl = pinn_flops(dims)
            roof = {"kernel": "k_pinn_chain* (K3, fp32 SIMT)", "bound": "alu",
                    "achieved": fl * evals / chain_s / 1e12,
                    "peak": ALU["fp32"] if ALU else n_sm * 128 * 2 * clk_mhz * 1e6 / 1e12, "unit": "TFLOP/s",
                    "peak_source": ALU["src"] if ALU else
                    "fp32 FMA pipe: %d SMs x 128 FMA/clk x 2 x %.0f MHz (nominal)" % (n_sm, clk_mhz),
                    "work_per_unit": "%.0f flop + %d tanh per point-eval" % (fl, sum(dims[1:-1])),
                    "launch_unit": "one coarse chain"}
            tr = ncu_traffic("k_pinn_chain")
        else:
            roof = {"kernel": "k_resident_chain (numerical G, fp64)", "bound": "alu",
                    "achieved": 9.0 * evals * p.coarse_steps / chain_s / 1e12,
                    "peak": ALU["fp64"] if ALU else n_sm * 64 * 2 * clk_mhz * 1e6 / 1e12, "unit": "TFLOP/s",
                    "peak_source": ALU["src"] if ALU else "fp64 pipe (nominal)",
                    "work_per_unit": "9 fp64 flop per point-step", "launch_unit": "one coarse chain"}
            tr = ncu_traffic("k_resident_chain")
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = tr["dram_bytes_per_launch"] if tr else None
    if tr:
        roof["traffic_source"] = tr.get("source")
    return roof


def c3_fine_sweep_roofline(parareal, synth, torch, stream, pk, pk_src, flush):
    """One Parareal iteration at C3 (2^20 points x 64 slices): its fine sweep (all 64 slices x 100
    steps) through the kernel the library picks (K2R, the grid-resident solver) and,
    beside it, forced through K2 (the HBM-streamed pass).  Roofline on SURVEY 8(d)'s algorithmic
    8 B per point-step from the CUDA-event phase time (median of 3, L2 flushed before each)."""
    p = synth.config("C3", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)

    def sweep_ms(fine_kernel):
        ctx = parareal.Context(p, stream=stream.cuda_stream)
        try:
            ctx.load_weights(synth.kaiming_net(synth.PINN_3x20, seed=0))
            ctx.set_option(parareal.OPT_USE_GRAPHS, 1)  # K2's ~200 pass launches replay as one graph
            ctx.set_option(parareal.OPT_FINE_KERNEL, fine_kernel)
            out = torch.empty((p.B, p.M), dtype=torch.float32, device="cuda")
            ctx.solve_device(out)
            ms = []
            for _ in range(3):
                flush.zero_()
                torch.cuda.synchronize()
                ms.append(ctx.solve_device(out)["ms_fine"])
            return statistics.median(ms)
        finally:
            ctx.close()

    with Clocks(torch.cuda.current_device()) as clk:
        t = sweep_ms(0) / 1e3      # auto: the grid-resident K2R at this size
    t_k2 = sweep_ms(2) / 1e3       # K2 forced
    pt_steps = float(p.M) * p.N * p.fine_steps
    ach = 8.0 * pt_steps / t / 1e9
    tr = ncu_traffic("k_fine_grid")
    tr2 = ncu_traffic("k_pass_res2")
    out = {"kernel": "k_fine_grid (K2R, grid-resident fine solver; state in registers, HBM once per slice)",
           "workload": "C3 fine sweep: 64 slices x 2^20 points x 100 IE steps",
           "bound": "hbm", "achieved": ach, "peak": float(pk["hbm_gbs"]), "unit": "GB/s",
           "frac": ach / float(pk["hbm_gbs"]), "peak_source": pk_src, "ms_per_sweep": t * 1e3,
           "point_steps_per_s": pt_steps / t,
           "work_per_unit": "8 B per point-step (SURVEY 8(d) algorithmic, single-pass design); K2R keeps the "
                            "state on chip, so this is the HBM-equivalent rate",
           "clocks": clk.summary(),
           "traffic": tr["dram_bytes_per_launch"] if tr else None,
           "traffic_unit": "bytes per sweep launch (ncu dram read+write; the whole sweep is one launch)",
           "k2": {"kernel": "k_pass_res2 (K2, persistent paired streamed pass)", "ms_per_sweep": t_k2 * 1e3,
                  "frac": 8.0 * pt_steps / t_k2 / 1e9 / float(pk["hbm_gbs"]),
                  "moved_bytes_frac": 16.0 * pt_steps / t_k2 / 1e9 / float(pk["hbm_gbs"]),
                  "moved_bytes_basis": "16 B per point-step: the two-pass kernel reads and writes fp32 state in both passes",
                  "traffic": tr2["dram_bytes_per_launch"] if tr2 else None,
                  "traffic_unit": "bytes per pass launch (one pass = 8 B per point)"}}
    if ALU:
        out["alu"] = {"achieved": 9.0 * pt_steps / t / 1e12, "peak": ALU["fp64"], "unit": "TFLOP/s",
                      "frac": 9.0 * pt_steps / t / 1e12 / ALU["fp64"],
                      "work_per_unit": "9 fp64 flop per point-step (the kernel issues ~2x: local run + rerun)"}
    return out


def training_run(synth):
    """The paper's PINN training (P:190 collocation counts: 5000 epochs at 1e-2 then 800
    at 1e-3, shuffled batches of 10 per epoch) of the 3x20 tanh net for the C2 market on this GPU,
    timed with CUDA events around the two pinn_train_epochs calls; plus the CPU oracle's time per
    Adam step on the same batch size (a bounded sample of 5 steps, numpy fp64, 1 process)."""
    import torch
    from paper_2303_03848_b200 import pinn_train
    mk = dict(K=1.0, sigma=0.2, r=0.05, T=1.0, L=4.0)
    sets = synth.collocation(mk, *synth.PAPER_COLLOCATION, seed=0)
    net0 = synth.pinn2_net([2, 20, 20, 20, 1], seed=0)
    st = torch.cuda.Stream()
    with pinn_train.Trainer(net0, mk, sets, batches=10, seed=0, stream=st.cuda_stream) as tr:
        l0 = tr.loss()
        tr.epochs(5, 1e-2, history=False)  # warm-up (graph capture, caches)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)                      # events on the trainer's stream (pinn_train_epochs syncs it)
        tr.epochs(5000, 1e-2, history=False)
        tr.epochs(800, 1e-3, history=False)
        e1.record(st)
        e1.synchronize()
        wall = e0.elapsed_time(e1) / 1e3
        l1 = tr.loss()
    steps = 5800 * 10
    pts = sum(synth.PAPER_COLLOCATION) / 10
    cpu_step = None
    try:
        from oracle import pinn_train as opt
        o = opt.Trainer(net0, mk, sets, batches=10, seed=0)
        o.gradient(0)
        t1 = time.perf_counter()
        for st in range(1, 6):
            o.gradient(st)
        cpu_step = (time.perf_counter() - t1) / 5
    except Exception:
        pass
    # algorithmic flops per point and step: forward jets 4 components x W^2 FMA per hidden layer,
    # the same again for h-bar and for the weight gradient (2 flop per FMA), plus the thin layers
    W, LHh = 20, 3
    flop_pt = 3 * 8 * W * W * (LHh - 1) + 3 * 8 * W * 3
    alu = alu_peaks()
    roof = {"kernel": "k_train_grad + k_adam (fp32 SIMT)", "bound": "alu",
            "achieved": flop_pt * pts / (wall / steps) / 1e12, "unit": "TFLOP/s",
            "peak": alu["fp32"] if alu else None, "peak_source": alu["src"] if alu else None,
            "work_per_unit": "%d flop per collocation point per step (3x20 net)" % flop_pt}
    roof["frac"] = roof["achieved"] / roof["peak"] if roof["peak"] else None
    return {"workload": "paper schedule: 5000 epochs lr 1e-2 + 800 epochs lr 1e-3, 10 shuffled batches/epoch, "
                        "N_f/N_b/N_exp = 100000/10000/10000 (P:190, P:210-211), 3x20 tanh, C2 market",
            "seconds": wall, "steps": steps, "us_per_step": 1e6 * wall / steps,
            "point_evals_per_s": steps * pts / wall, "loss_initial": list(map(float, l0)),
            "loss_final": list(map(float, l1)),
            "paper_context": "P:212: 'around 30 minutes' for the paper's 10x50 ReLU net (other hardware)",
            "cpu_oracle_s_per_step": cpu_step,
            "cpu_oracle_sample": "5 gradient evaluations of the numpy fp64 training oracle on the same batch (1 process)",
            "roofline": roof}


CONVERGED_TOL = {"C1": 3e-5, "C2": 1e-5, "C3": 3e-5}  # Q18-valid tolerances


def converged_run(args, parareal, synth, torch, stream, flush):
    """Converged-K speedup (fixed K=3 AND converged K): the same grid with the
    numerical coarse G (IE, 1 step/slice), tol from CONVERGED_TOL, max_iter = N; blocking schedule
    (a tolerance needs the host's stop decision between iterations).  Median and mean ± std of 5
    solves (CUDA events on the launching stream), and the GPU serial fine solve of the same grid."""
    tol = CONVERGED_TOL[args.config.upper()]
    p = synth.config(args.config, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1, tol=tol,
                     fine_theta=args.fine_theta)
    p = p.replace(max_iter=p.N)
    ctx = parareal.Context(p, stream=stream.cuda_stream)
    try:
        out = torch.empty((p.B, p.M), dtype=torch.float32, device="cuda")
        rep = ctx.solve_device(out)
        ms = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = ctx.solve_device(out)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        sf = []
        for _ in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            sf.append(ctx.serial_fine_device(out))
        serial = statistics.median(sf)
        return {"coarse": "implicit Euler, 1 step/slice", "tol": tol, "iterations": rep["iterations"],
                "converged": rep["converged"], "delta": [float(d) for d in rep["delta"]],
                "ms_per_solve": step_stats(ms), "serial_fine_ms": serial,
                "speedup_vs_serial_fine": serial / statistics.median(ms),
                "value": work_units(p) / (statistics.median(ms) / 1e3), "unit": UNIT}
    finally:
        ctx.close()


# --------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    from paper_2303_03848_b200 import parareal, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print("warning: --gpus %d but WORLD_SIZE %d" % (args.gpus, world), file=sys.stderr)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p = problem_for(args)
    # C4 (the batched portfolio) shards its independent instances across the GPUs (SURVEY §8(e):
    # no data-path collective; fixed K, so no δ all-reduce either): each rank solves its B/R
    # instances as a one-GPU problem.  The other configs shard the time slices (NCCL chain).
    shard_inst = args.config.upper() == "C4" and world > 1
    if shard_inst:
        if p.B % world:
            raise SystemExit("B=%d not divisible by %d GPUs" % (p.B, world))
        p_run, ctx_world, ctx_rank = synth.shard_instances(p, rank, world), 1, 0
    else:
        if p.N % world:
            raise SystemExit("N=%d not divisible by %d GPUs" % (p.N, world))
        p_run, ctx_world, ctx_rank = p, world, rank
    net = synth.kaiming_net(pinn_dims(args), seed=0)
    nccl_id = None
    if ctx_world > 1:
        obj = [parareal.get_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    # one dedicated stream for everything timed: the L2 flush, the CUDA events and the library's
    # kernels (torch's default stream is the legacy NULL stream; a context given NULL would create
    # its own non-blocking stream, which the events on the NULL stream would not order with)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = parareal.Context(p_run, rank=ctx_rank, world=ctx_world, device=local, nccl_id=nccl_id,
                           stream=stream.cuda_stream)
    if p.coarse == synth.COARSE_PINN:
        ctx.load_weights(net, precision=PREC_CODE[args.pinn_prec])
    ws = torch.empty(ctx.workspace_bytes(), dtype=torch.uint8, device="cuda")
    ctx.bind_workspace(ws)
    # fixed-K single-GPU solves replay one CUDA graph; in the timed loop the lean, stream-ordered
    # replay (no phase-timing nodes, returns once enqueued), so the CUDA events bracket device time
    # only; the phase times come from a few instrumented replays afterwards
    graph_timed, graph_phases = (0, 0) if args.no_graphs else (2, 1)
    ctx.set_option(parareal.OPT_USE_GRAPHS, graph_timed)
    out = torch.empty((p_run.B, p.M), dtype=torch.float32, device="cuda")
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        ctx.solve_device(out)
    torch.cuda.synchronize()
    # ---------------- timed region: device time of K solves (events on the launching stream)
    step_ms, reps = [], []
    barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            reps.append(ctx.solve_device(out))
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    barrier()
    if graph_timed != graph_phases:  # instrumented solves for the phase times
        ctx.set_option(parareal.OPT_USE_GRAPHS, graph_phases)
        ctx.solve_device(out)
        reps = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            torch.cuda.synchronize()
            reps.append(ctx.solve_device(out))
    total = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    total_ms = float(total.item())
    ms_step = total_ms / args.steps
    value = work_units(p) * args.steps / (total_ms / 1e3)
    launches = int(reps[0]["kernel_launches"]) * args.steps  # per solve (the same kernels every step)
    # ---------------- serial fine baseline (one GPU) and Eq. (8) context
    serial_ms = None
    if rank == 0:
        for _ in range(2):
            ctx.serial_fine_device(out)
        sm = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            torch.cuda.synchronize()
            sm.append(ctx.serial_fine_device(out))
        serial_ms = statistics.median(sm)
    K = p.max_iter
    ph = {k: statistics.median([r[k] for r in reps]) for k in ("ms_fine", "ms_coarse", "ms_comm", "ms_setup",
                                                               "ms_total")}
    # pipelined schedule: its phases overlap (reported as one span); the blocking schedule's phase
    # times (a few solves) give Eq. (8)'s c_c, c_f and the pipelining gain
    ph_block, block_ms = ph, None
    if ph["ms_fine"] == ph["ms_coarse"] and ctx_world == 1:
        ctx.set_option(parareal.OPT_PIPELINE, 1)
        ctx.solve_device(out)
        breps = []
        for _ in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            breps.append(ctx.solve_device(out))
        ph_block = {k: statistics.median([r[k] for r in breps]) for k in ph}
        block_ms = ph_block["ms_total"]
        ctx.set_option(parareal.OPT_PIPELINE, 0)
    # ---------------- roofline of the dominant kernel (per-launch average, events per phase)
    pk, pk_src = peaks()
    global ALU
    ALU = alu_peaks()
    clk_mhz = float(pk.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    roof = roofline(p_run, ph, K, ctx_world, ctx_rank, pk, pk_src, clk_mhz, n_sm, synth, dims=pinn_dims(args),
                    tc_prec=None if args.pinn_prec == "fp32" else args.pinn_prec)
    # ---------------- north-star gate: the HBM-streamed fine sweep (K2) at the C3 grid, measured
    # live in the same run (one fine sweep over 64 slices x 2^20 points x 100 steps)
    fine_c3 = None
    if rank == 0 and world == 1 and not args.no_c3_sweep and args.config != "C3":
        fine_c3 = c3_fine_sweep_roofline(parareal, synth, torch, stream, pk, pk_src, flush)
    # ---------------- converged-K run: iterate until δ^k < tol (numerical G; with Kaiming-random PINN
    # weights Parareal only terminates at k = N, so the tolerance run uses the coarse IE propagator)
    converged = None
    if rank == 0 and world == 1 and args.config.upper() in CONVERGED_TOL:
        converged = converged_run(args, parareal, synth, torch, stream, flush)
    # ---------------- NEXT-3: PINN training on the GPU (the paper's sets and schedule)
    training = None
    if rank == 0 and world == 1 and not args.no_training:
        training = training_run(synth)
    # ---------------- e2e through the host-buffer ABI call (pinned H2D of V_T, D2H of V_0)
    e2e = None
    if not args.no_e2e:
        has_vt = ctx_rank == 0  # (slice sharding: rank 0 owns U_0; instance sharding: every rank)
        vt_host = torch.from_numpy(ctx.initial_state()).pin_memory() if has_vt else None
        v0_host = torch.empty((p_run.B, p.M), dtype=torch.float32).pin_memory()
        ctx.solve_host_ptrs(vt_host.data_ptr() if has_vt else None, v0_host.data_ptr())
        barrier()
        torch.cuda.synchronize()
        ems = []
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.solve_host_ptrs(vt_host.data_ptr() if has_vt else None, v0_host.data_ptr(), report=False)
            e1.record(stream)
            e1.synchronize()
            ems.append(e0.elapsed_time(e1))
        et = torch.tensor([sum(ems)], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": work_units(p) * args.steps / (float(et.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 4 * p.B * p.M, "d2h_bytes_per_step": 4 * p.B * p.M}
    # ---------------- CPU oracle baseline (rank 0, N=1 only)
    cpu = cpu_threaded = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from paper_2303_03848_b200 import synth as S
        netc = net if p.coarse == S.COARSE_PINN else None
        per, runs, cores = cpu_oracle_run(p, netc, budget_s=10.0, max_runs=20)
        cpu = {"value": work_units(p) / per, "unit": UNIT, "cores": cores, "kind": "oracle",
               "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
               "sample": "full %s workload, %d serial fp64 oracle solves (%.3f s each)" % (args.config, runs, per)}
        nth = max(1, min(p.N, os.cpu_count() or 1))
        per_t, runs_t, _ = cpu_oracle_run(p, netc, budget_s=10.0, max_runs=20, threads=nth)
        cpu_threaded = {"value": work_units(p) / per_t, "unit": UNIT, "cores": nth, "kind": "oracle, threaded fine sweep",
                        "sample": "full %s workload, %d fp64 oracle solves with the fine sweep on %d std::threads "
                                  "(%.3f s each; bitwise the serial result)" % (args.config, runs_t, nth, per_t)}
    if rank == 0:
        from paper_2303_03848_b200 import report
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32 state / f64 implicit solves / f32 PINN",
                "data": "synthetic (payoff initial state, Kaiming-random PINN weights seed 0)",
                "config": dict(config_dict(args, p), **({"parallelism": "instances/%d (B/R per GPU, no exchange)" % world}
                                                        if shard_inst else {})),
                "speedup_vs_serial_fine": (serial_ms / ms_step) if serial_ms else None,
                "serial_fine_ms": serial_ms,
                "phases_ms": ph,
                # throughputs of the two phases, from the BLOCKING schedule's phase times (in the
                # pipelined kernel the phases overlap and have no separate duration)
                "pinn_evals_per_s_coarse_phase": (float(p.B) * p.M * sum(p.N - k for k in range(0, K + 1))
                                                  / (ph_block["ms_coarse"] / 1e3))
                if p.coarse == synth.COARSE_PINN and ph_block["ms_coarse"] > 0 else None,
                "fine_point_steps_per_s_fine_phase": float(p.B) * p.M * p.fine_steps
                * sum(p.N - k + 1 for k in range(1, K + 1)) / (ph_block["ms_fine"] / 1e3)
                if ph_block["ms_fine"] > 0 else None,
                "phase_basis": "blocking schedule (PR_OPT_PIPELINE=1) phase times" if block_ms is not None
                else "this schedule's phase times",
                "step_ms_stats": step_stats(step_ms),
                "eq8_bound_context": None,
                "roofline": roof, "roofline_fine_sweep_c3": fine_c3, "converged_K_run": converged,
                "pinn_training": training,
                "cpu_baseline": cpu,
                "cpu_baseline_threaded": cpu_threaded, "e2e": e2e,
                "gpu_launches": launches,
                "clocks": clk.summary()}
        if shard_inst:
            line["speedup_basis"] = ("per GPU: the serial fine solve of one rank's B/R instances vs the Parareal "
                                     "step (every rank solves its own instances)")
        line["schedule"] = "pipelined" if block_ms is not None else "blocking"
        if block_ms is not None:
            line["blocking_schedule_ms_per_solve"] = block_ms
        if serial_ms and ph_block["ms_coarse"] > 0:
            c_f = serial_ms / p.N
            c_c = ph_block["ms_coarse"] / (K + 1) / p.N
            line["eq8_bound_context"] = {"c_c_ms": c_c, "c_f_ms": c_f,
                                         "pipelined": report.speedup_bound(K, p.N, c_c / c_f),
                                         "blocking": report.speedup_bound_blocking(K, p.N, c_c / c_f)}
        print(json.dumps(line))
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
