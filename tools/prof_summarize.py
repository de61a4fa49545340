"""Summarise the ncu captures of tools/prof_capture.sh (gpurun_out/) into
profiles/: a markdown table of the key counters per captured kernel, the
per-launch DRAM traffic of the dominant kernel (read by bench.py for the
roofline's `traffic`), and the launch-list shares of one training step.

    python tools/prof_summarize.py [--round r01]
"""
from __future__ import annotations

import argparse
import csv
import glob
import io
import json
import os
import re
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "tensor_imma_pct": "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "inst_M": "smsp__inst_executed.sum",
}


def raw_rows(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": re.sub(r"\(.*", "", d.get("Kernel Name", "?"))[:90]}
        for k, m in KEYS.items():
            v = d.get(m)
            if v in (None, ""):
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            unit = u.get(m, "")
            if k.endswith("_MB"):
                x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1e-6)
            if k == "duration_us" and unit == "ms":
                x *= 1e3
            if k == "duration_us" and unit == "ns":
                x *= 1e-3
            if k == "inst_M":
                x /= 1e6
            rec[k] = round(x, 3)
        out.append(rec)
    return out


def launches(path):
    if not os.path.exists(path):
        return None
    if path.endswith(".gz"):
        import gzip
        lines = gzip.open(path, "rt").read().splitlines()
    else:
        lines = open(path).read().splitlines()
    start = next((i for i, l in enumerate(lines) if l.startswith('"ID"')), None)
    if start is None:
        return None
    rows = list(csv.DictReader(lines[start:]))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        name = r["Kernel Name"]
        key = ("libhlq: " + re.sub(r"\(.*", "", name).split("::")[-1][:48]) if "hlq::" in name else \
            "torch/cuBLAS/cuDNN: " + re.sub(r"\(.*", "", name).replace("void ", "")[:60]
        agg[key][0] += 1
        agg[key][1] += us
        total += us
    return total, agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--out", default=PROF, help="where the summaries go (profiles/ by default)")
    ap.add_argument("--reps", default=OUT, help="directory holding the prof_*.ncu-rep files")
    ap.add_argument("--launches", default=os.path.join(OUT, "launches.csv"))
    a = ap.parse_args()
    prof = a.out
    os.makedirs(prof, exist_ok=True)
    md = [f"# {a.round} ncu summary (B200, sm_100a, `--clock-control none`)\n",
          "Captured by `tools/prof_capture.sh` under gpurun; numbers under a profiler are not bench values --",
          "durations are single serialised launches, the counters are what matter.\n"]
    summary = {}
    reps = sorted(glob.glob(os.path.join(a.reps, "prof_*.ncu-rep")))
    for rep in reps:
        tag = os.path.basename(rep)[5:-8]
        rows = raw_rows(rep)
        summary[tag] = rows
        if not rows:
            continue
        md.append(f"## {tag}\n")
        cols = ["kernel"] + [k for k in KEYS if any(k in r for r in rows)]
        md.append("| " + " | ".join(cols) + " |")
        md.append("|" + "---|" * len(cols))
        for r in rows:
            md.append("| " + " | ".join(str(r.get(c, "")) for c in cols) + " |")
        md.append("")
    la = launches(a.launches)
    if la:
        total, agg = la
        # the capture spans several training steps (bench.py warm-up, timed, traced, e2e);
        # the batched weight-codes kernel runs exactly once per step
        steps = max(1, next((v[0] for k, v in agg.items() if "weight_codes" in k), 1))
        md.append("## One ViT-B/16 HLQ training step: launch list (ncu, serialised, cold L2)\n")
        md.append(f"Captured over {steps} training steps of `bench.py --steps 1 --warmup 1 --no-extras`; "
                  "per-step averages below (model construction kernels included in the torch rows).\n")
        hlq = sum(v[1] for k, v in agg.items() if k.startswith("libhlq"))
        md.append(f"Kernel time per step {total / steps / 1e3:.2f} ms; libhlq kernels {hlq / steps / 1e3:.2f} ms "
                  f"({100 * hlq / total:.1f} %).\n")
        md.append("| kernel | launches/step | us/step | share |")
        md.append("|---|---|---|---|")
        for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
            md.append(f"| {k} | {n / steps:.1f} | {us / steps:.1f} | {100 * us / total:.1f} % |")
        md.append("")
    open(os.path.join(prof, f"{a.round}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(summary, open(os.path.join(prof, f"{a.round}_ncu_counters.json"), "w"), indent=1)
    # per-launch DRAM traffic of the dominant kernel class (the fused transform) for bench.py
    dual = summary.get("dual") or []
    if dual:
        r = dual[0]
        traffic = {"kernel": r["kernel"], "workload": "ViT-B/16 fc1 gy (128x197x3072 bf16), dual transform",
                   "key": "transform:dual:25216x3072:bfloat16",
                   "dram_bytes_per_launch": round((r.get("dram_read_MB", 0) + r.get("dram_write_MB", 0)) * 1e6),
                   "algorithmic_bytes_per_launch": int(128 * 197 * 3072 * 2 + 128 * 197 * 3072 + 3072 * 13312),
                   "source": f"profiles/{a.round}_ncu_counters.json"}
        json.dump(traffic, open(os.path.join(prof, f"{a.round}_traffic.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
