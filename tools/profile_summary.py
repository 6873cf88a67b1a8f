#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (tracked).

    python tools/profile_summary.py --launches gpurun_out/launches_c4.csv \
        --full gpurun_out/prof.ncu-rep --cells 16777216 --workload C4s --out profiles/r1

Writes <out>_launches.md (per-kernel share of the launch list),
<out>_full.md (key counters of the --set full capture) and updates
profiles/traffic.json (DRAM bytes per launch of the step kernel, used by
bench.py's roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (registers), CTAs"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / instruction"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread ops"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread ops"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread ops"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait / issue"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
     "stall: no_instruction / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
     "stall: short_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
     "stall: branch_resolving / issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "stall: long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
     "stall: math_pipe_throttle / issue"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
                 "msecond": 1.0}.get(unit, 1.0)
        name = r[ik].split("(")[0]
        tot[name] += v * scale
        cnt[name] += 1
    return tot, cnt


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for k, label in KEYS:
        if k in hdr:
            i = hdr.index(k)
            res[k] = (label, vals[i], units[i])
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    return name, res


def opcode_mix(rep):
    """Dynamic mix: executed warp instructions per SASS opcode (ncu's
    sass__inst_executed_per_opcode, instance names = opcodes)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--metrics",
                          "sass__inst_executed_per_opcode", "--print-metric-instances", "details"],
                         capture_output=True, text=True).stdout
    flat = " ".join(out.split())
    i = flat.find("sass__inst_executed_per_opcode")
    if i < 0 or "(" not in flat[i:]:
        return []
    body = flat[flat.index("(", i) + 1:]
    body = body[:body.index(")")]
    mix = []
    for item in body.split(";"):
        if ":" in item:
            op, v = item.split(":")
            mix.append((op.strip(), int(v.strip())))
    return sorted(mix, key=lambda x: -x[1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--cells", type=float)
    ap.add_argument("--workload", default="C4s")
    ap.add_argument("--out", required=True)
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    if a.launches:
        tot, cnt = launches(a.launches)
        s = sum(tot.values())
        with open(a.out + "_launches.md", "w") as fh:
            fh.write(f"# Launch list ({os.path.basename(a.launches)})\n\n")
            if a.command:
                fh.write(f"Command: `{a.command}`\n\n")
            fh.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, "
                     "serialised launches: compare shares, not absolute times).\n\n")
            fh.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
            for k, v in sorted(tot.items(), key=lambda x: -x[1]):
                fh.write(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / s:.1f}% |\n")
    if a.full:
        name, res = full(a.full)
        with open(a.out + "_full.md", "w") as fh:
            fh.write(f"# ncu --set full: `{name[:90]}`\n\nWorkload {a.workload}")
            if a.cells:
                fh.write(f", {int(a.cells)} cells per launch")
            fh.write("\n\n| counter | value | unit |\n|---|---|---|\n")
            for k, (label, v, u) in res.items():
                fh.write(f"| {label} (`{k}`) | {v} | {u} |\n")
            if a.cells:
                rd = float(res["dram__bytes_read.sum"][1])
                wr = float(res["dram__bytes_write.sum"][1])
                unit = res["dram__bytes_read.sum"][2]
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                b = (rd + wr) * mult
                fh.write(f"\nDRAM bytes per cell-update: {b / a.cells:.1f} "
                         f"(algorithmic: 64)\n")
                tp = os.path.join(os.path.dirname(a.out) or ".", "traffic.json")
                tj = json.load(open(tp)) if os.path.exists(tp) else {}
                entry = {"dram_bytes_per_launch": b, "cells": a.cells,
                         "source": os.path.basename(a.out) + "_full.md"}
                tj[a.workload] = entry
                json.dump(tj, open(tp, "w"), indent=1)
            mix = opcode_mix(a.full)
            if mix and a.cells:
                # FP64-pipe thread instructions per cell-update (DFMA/DMUL/DADD/DSETP),
                # for bench.py's roofline_fp64 (the active path's binding roof)
                k = "smsp__thread_inst_executed_per_inst_executed.ratio"
                lanes = float(res[k][1]) if k in res else 32.0
                fp = sum(v for op, v in mix if op in ("DFMA", "DMUL", "DADD", "DSETP"))
                tp = os.path.join(os.path.dirname(a.out) or ".", "traffic.json")
                tj = json.load(open(tp)) if os.path.exists(tp) else {}
                tj.setdefault(a.workload, {})["fp64_pipe_inst_per_cell"] = lanes * fp / a.cells
                json.dump(tj, open(tp, "w"), indent=1)
            if mix:
                tot = sum(v for _, v in mix)
                fp64 = sum(v for op, v in mix if op in ("DFMA", "DMUL", "DADD", "DSETP"))
                k = "smsp__thread_inst_executed_per_inst_executed.ratio"
                lanes = float(res[k][1]) if k in res else 32.0
                fh.write("\nDynamic instruction mix (executed warp instructions per SASS opcode, "
                         "`sass__inst_executed_per_opcode`)")
                if a.cells:
                    fh.write(f"; per cell-update = count x {lanes:.2f} active lanes per warp "
                             f"instruction / {int(a.cells)} cells (thread instructions)")
                fh.write(f".  FP64 pipe (DFMA+DMUL+DADD+DSETP): {100 * fp64 / tot:.1f}% of "
                         "all instructions.\n\n| opcode | warp instructions | share |"
                         + (" per cell-update |" if a.cells else "") + "\n|---|---|---|"
                         + ("---|" if a.cells else "") + "\n")
                for op, v in mix[:24]:
                    fh.write(f"| {op} | {v} | {100 * v / tot:.1f}% |"
                             + (f" {lanes * v / a.cells:.1f} |" if a.cells else "") + "\n")


if __name__ == "__main__":
    main()
