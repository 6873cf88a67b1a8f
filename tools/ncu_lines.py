#!/usr/bin/env python
"""Attribute an ncu source-page profile to CUDA source lines.

    python tools/ncu_lines.py PROFILE.ncu-rep KERNEL_SUBSTRING LIB.so [TU_SUBSTRING]

Joins ncu's per-SASS-instruction counters (--page source --print-source=sass)
with `nvdisasm -g` line info of the same binary (instruction order), then
prints the hottest source lines by executed warp instructions and by stall
samples.  The .so must be the exact build that was profiled.
"""
from __future__ import annotations

import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def ncu_rows(rep: str, kernel: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')
    for b in blocks[1:]:
        head, _, body = b.partition("\n")
        if kernel not in head:
            continue
        rows = list(csv.reader(io.StringIO(body)))
        hdr = rows[0]
        return hdr, rows[1:]
    raise SystemExit(f"kernel {kernel} not in profile")


def sass_lines(lib: str, kernel_mangled_part: str, tu: str):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d,
                   capture_output=True)
    cubins = [f for f in os.listdir(d) if f.endswith(".cubin") and tu in f]
    for cb in cubins:
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cb)],
                             capture_output=True, text=True).stdout
        secs = re.split(r"\n(?=\.text\.)", dis)
        for sec in secs:
            if not sec.startswith(".text.") or kernel_mangled_part not in sec.split(":")[0]:
                continue
            cur = "?"
            out = []
            for line in sec.split("\n"):
                m = re.search(r'//## File "([^"]+)", line (\d+)', line)
                if m:
                    cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                    continue
                if re.search(r"/\*[0-9a-f]{4,}\*/", line):
                    out.append(cur)
            return out
    raise SystemExit("kernel not found in cubin")


def main():
    rep, kernel, lib = sys.argv[1:4]
    tu = sys.argv[4] if len(sys.argv) > 4 else "fast"
    hdr, rows = ncu_rows(rep, kernel)
    ie = hdr.index("Instructions Executed")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    isrc = hdr.index("Source")
    mangled = "step2d_kernel" if "step2d" in kernel else kernel
    lines = sass_lines(lib, mangled, tu)
    n = min(len(lines), len(rows))
    if len(lines) != len(rows):
        print(f"warning: {len(lines)} disassembled vs {len(rows)} profiled instructions")
    inst = collections.Counter()
    stall = collections.Counter()
    tot_i = tot_s = 0.0
    for k in range(n):
        e = float(rows[k][ie] or 0)
        s = float(rows[k][iss] or 0)
        inst[lines[k]] += e
        stall[lines[k]] += s
        tot_i += e
        tot_s += s
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
    print("by stall samples:")
    for ln, v in stall.most_common(40):
        print(f"  {ln:28s} stall {100 * v / tot_s:5.2f}%  inst {100 * inst[ln] / tot_i:5.2f}%")


if __name__ == "__main__":
    main()
