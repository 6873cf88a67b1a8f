#!/usr/bin/env python
"""Top CUDA source lines of a profile by executed instructions (with opcode mix)."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines as N
rep, lib, tu = sys.argv[1], sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "fast")
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
hdr, rows = N.ncu_rows(rep, "step2d")
lines = N.sass_lines(lib, os.environ.get("SILT_NCU_KERNEL", "step2d_kernel"), tu)
ie, isrc, iss = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
inst, stall, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
for k in range(min(len(lines), len(rows))):
    e = float(rows[k][ie] or 0); s = float(rows[k][iss] or 0)
    inst[lines[k]] += e; stall[lines[k]] += s
    op = rows[k][isrc].split()
    o = op[1] if op and op[0].startswith('@') else (op[0] if op else '?')
    ops[lines[k]][o.split('.')[0]] += e
ti, ts = sum(inst.values()), sum(stall.values())
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1307_0491_b200", "csrc")
src = {f: open(os.path.join(root, f)).read().split("\n") for f in os.listdir(root) if f.endswith((".cuh", ".h"))}
for ln, v in inst.most_common(n):
    f, _, l = ln.partition(":")
    text = src[f][int(l) - 1].strip()[:64] if f in src else ""
    top = ",".join(f"{o}{int(c / v * 100)}" for o, c in ops[ln].most_common(3))
    print(f"{v / ti * 100:5.2f}% st{stall[ln] / ts * 100:5.2f}% {ln:24s} {top:26s} {text}")
