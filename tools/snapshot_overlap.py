#!/usr/bin/env python
"""Wall time of a run with snapshots: synchronous gather vs asynchronous capture.

    python tools/snapshot_overlap.py [--n 16384] [--steps 200] [--snaps 4]

Runs the C4-type dune (n x n, A_g = 0.001) for --steps steps with --snaps
snapshot times spread over the run, once with synchronous snapshots (pause,
download, callback, resume) and once with asynchronous captures (the copy to
pinned memory overlaps the following steps).  The callback does what a writer
would start with: it touches every value (a checksum).  Prints one JSON line.
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
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1307_0491_b200 import native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--snaps", type=int, default=4)
    a = ap.parse_args()
    p = bench.build_global_problem(a.workload, 1)
    full = bench.device_initial_rows(a.workload, p, 0, p.ny, torch.device("cuda"))
    torch.cuda.synchronize()
    # time of step `steps` from a probe run, to place the snapshots inside the run
    s = native.Solver(p)
    s.upload_device(full.data_ptr())
    s.begin(max_steps=a.steps)
    st = s.run(batch=64)
    t_run = st.t
    s.close()
    snaps = [t_run * (k + 1) / (a.snaps + 1) for k in range(a.snaps)]
    out = {"workload": a.workload, "cells": p.nx * p.ny, "steps": a.steps, "snapshots": snaps}
    for mode in (False, True):
        s = native.Solver(p)
        s.upload_device(full.data_ptr())
        s.begin(max_steps=a.steps + a.snaps, snapshots=snaps)
        sums = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = s.run(batch=32, on_snapshot=lambda t, f: sums.append(float(np.sum(f[..., 0]))),
                   async_snapshots=mode)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        s.close()
        out["async" if mode else "sync"] = {"wall_s": wall, "steps": st.steps, "sum_h": sums}
    out["saved_s"] = out["sync"]["wall_s"] - out["async"]["wall_s"]
    assert out["sync"]["sum_h"] == out["async"]["sum_h"]
    # CSV snapshots (device formatter) to /dev/null: between steps vs in the background
    for mode in ("csv_sync", "csv_async"):
        s = native.Solver(p)
        s.upload_device(full.data_ptr())
        s.write_snapshot(0.0, "/dev/null")  # CSV context warm-up
        s.begin(max_steps=a.steps + a.snaps, snapshots=snaps)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode == "csv_async":
            st = s.run_csv("/dev/null%.0s", batch=32)  # every snapshot to /dev/null
        else:
            while True:
                s.step(32)
                st = s.status()
                if st.state == 2:
                    s.write_snapshot(st.t, "/dev/null")
                    s.resume()
                    continue
                if st.state == 1:
                    break
        torch.cuda.synchronize()
        out[mode] = {"wall_s": time.perf_counter() - t0, "steps": st.steps}
        s.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
