"""Proxy for two pieces per rank: the step time of ONE contiguous
strip that holds 1/N of the grid's rows with 1/N of the mound's rows in it (a
far-field band plus a mound band, adjacent), against T1 / N.  If a launch that
mixes hot and quiescent row blocks runs at the one-GPU pace, a rank stepping
one mound piece and one far-field piece in one launch would too.

    python tools/mix_probe.py [--workload C4] [--ns 4,8]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench  # noqa: E402
from strip_times import strip_ms  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--ns", default="4,8")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    p = bench.build_global_problem(a.workload, 1)
    full = bench.device_initial_rows(a.workload, p, 0, p.ny, torch.device("cuda"))
    t1 = strip_ms(p, full, 0, p.ny, a.steps, a.warmup)
    # mound rows of the dune workloads: bump on y in [400, 600] m, waves included
    # the hot band is taken as [0.38, 0.62] of the rows
    lo, hi = int(0.38 * p.ny), int(0.62 * p.ny)
    print(f"T1 {t1:.3f} ms; hot band rows [{lo}, {hi})")
    for n in map(int, a.ns.split(",")):
        rows = p.ny // n
        hot = (hi - lo) // n
        j0 = lo - (rows - hot)  # far-field rows below, then 1/n of the hot band
        t = strip_ms(p, full, j0, rows, a.steps, a.warmup)
        t_hot = strip_ms(p, full, lo + (hi - lo) // 2 - rows // 2, rows, a.steps, a.warmup)
        print(f"N={n}: mixed strip [{j0}, {j0 + rows}) {t:.3f} ms, efficiency {t1 / (n * t):.2f}; "
              f"all-mound strip {t_hot:.3f} ms ({t1 / (n * t_hot):.2f})")


if __name__ == "__main__":
    main()
