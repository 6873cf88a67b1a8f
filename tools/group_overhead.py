#!/usr/bin/env python
"""Per-step time of the in-process strip group (silt_group, the C++ drop-in's
run_parallel) on one GPU: py strips of a workload, direct mode (edge rows
stored by the step kernels into the neighbours' buffers, maxima pushed by
remote atomics, event ordering) vs copy mode (SILT_GROUP_DIRECT=0: row copies
and a reduction kernel per step).

    SILT_GROUP_DIRECT=0|1 python tools/group_overhead.py [--workload C3] [--py 1,2,4,8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1307_0491_b200 import scenarios  # noqa: E402
from paper_1307_0491_b200.distributed import LocalStripGroup  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--py", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    p, init, _ = scenarios.dune_2d(a.n)
    out = {"n": a.n, "direct": os.environ.get("SILT_GROUP_DIRECT", "1"), "ms_per_step": {}}
    for py in [int(x) for x in a.py.split(",")]:
        g = LocalStripGroup(p, py, devices=(0,))
        g.upload(init)
        g.begin(max_steps=a.steps + 20)
        g.step(20)
        g.status()
        t0 = time.perf_counter()
        g.step(a.steps)
        g.status()
        out["ms_per_step"][py] = (time.perf_counter() - t0) * 1e3 / a.steps
        g.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
