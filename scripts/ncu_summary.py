#!/usr/bin/env python
"""Summarise `ncu --set full` captures (.ncu-rep) into profiles/.

  python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep [...] --out profiles/r01_ncu_summary.md
      [--traffic profiles/ncu_traffic.json]

Per launch: duration, DRAM bytes (read+write), DRAM/L2/issue utilisation, pipe utilisation,
occupancy, registers and the top warp-stall reasons.  --traffic merges
dram__bytes_read.sum + dram__bytes_write.sum per kernel into the JSON bench.py reads for the
roofline `traffic` field.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"), ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pipe_%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
        ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
              "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1.0}


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:] if r]


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def summarise(rep):
    res = []
    for d, u in raw(rep):
        rec = {"kernel": d.get("Kernel Name", "?"), "source": os.path.basename(rep)}
        for k, name in KEYS:
            if k in d:
                v = num(d[k])
                sc = UNIT_SCALE.get(u.get(k, ""), 1)
                rec[name] = v * sc if v is not None and name in ("duration", "dram_read", "dram_write") else v
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                x = num(v)
                if x:
                    stalls.append((x, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(x for x, _ in stalls) or 1
        rec["stalls"] = ", ".join("%s %.0f%%" % (n, 100 * x / tot) for x, n in sorted(stalls, reverse=True)[:5])
        res.append(rec)
    return res


def measured_hbm_gbs():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    ap.add_argument("--title", default="ncu --set full captures")
    args = ap.parse_args()
    recs = [r for rep in args.reps for r in summarise(rep)]
    lines = ["# %s" % args.title, "",
             "DRAM GB/s = dram__bytes (read+write) / gpu__time_duration of the launch under ncu; "
             "'of meas.' divides by the measured copy bandwidth in MEASURED_PEAKS.json (%s GB/s)." % measured_hbm_gbs(), "",
             "| kernel | source | time (us) | DRAM R+W (MB) | DRAM GB/s | of meas. | DRAM % | L2 % | issue % | warps % | fma % | fp64 % | xu % | tensor % | regs | grid | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    hbm = measured_hbm_gbs()
    for r in recs:
        f = lambda k, s=1, p=1: ("%.*f" % (p, r[k] * s)) if r.get(k) is not None else "-"
        dram = (r.get("dram_read") or 0) + (r.get("dram_write") or 0)
        gbs = dram / r["duration"] / 1e9 if r.get("duration") else None
        lines.append("| %s | %s | %s | %.2f | %s | %s | %s | %s | %s | %s | %s | %s | %s | %s | %s | %s | %s |" % (
            r["kernel"][:60], r["source"], f("duration", 1e6), dram / 1e6,
            "%.0f" % gbs if gbs is not None else "-", "%.2f" % (gbs / hbm) if (gbs and hbm) else "-",
            f("dram_%"), f("l2_%"), f("issue_%"),
            f("warps_active_%"), f("fma_pipe_%"), f("fp64_pipe_%"), f("xu_pipe_%"), f("tensor_pipe_%"),
            f("regs", 1, 0), f("grid", 1, 0), r["stalls"]))
    with open(args.out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if args.traffic:
        try:
            with open(args.traffic) as fh:
                tj = json.load(fh)
        except Exception:
            tj = {"_doc": "dram__bytes_read.sum + dram__bytes_write.sum per launch from ncu --set full "
                          "(scripts/ncu_summary.py); read by bench.py for roofline.traffic", "kernels": {}}
        for r in recs:
            name = r["kernel"].split("(")[0].replace("void ", "").replace("pr::", "").strip()
            tj["kernels"][name] = {"dram_bytes_per_launch": (r.get("dram_read") or 0) + (r.get("dram_write") or 0),
                                   "duration_s_under_ncu": r.get("duration"), "source": r["source"]}
        with open(args.traffic, "w") as fh:
            json.dump(tj, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
