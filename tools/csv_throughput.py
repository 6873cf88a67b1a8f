#!/usr/bin/env python
"""Snapshot CSV throughput: the device writer vs the reference's snapshot_to_string.

    python tools/csv_throughput.py [--workload C4] [--sink /dev/null]

The device writer formats the solver's state (C4: 268 M cells) and streams
the bytes to --sink; the reference (oracle/_ref, else the restatement) formats
a 96-row band of the same field on one host core.  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1307_0491_b200 import abi, native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--sink", default="/dev/null")
    a = ap.parse_args()
    p = bench.build_global_problem(a.workload, 1)
    full = bench.device_initial_rows(a.workload, p, 0, p.ny, torch.device("cuda"))
    torch.cuda.synchronize()
    s = native.Solver(p)
    s.upload_device(full.data_ptr())
    s.write_snapshot(0.0, a.sink)  # warm-up (context, pinned buffers)
    t0 = time.perf_counter()
    nbytes = s.write_snapshot(12.5, a.sink)
    gpu_s = time.perf_counter() - t0
    s.close()
    cells = p.nx * p.ny
    # reference on a band of rows (host)
    import oracle as O
    R = O.reference() if O.have_reference() else O.restatement()
    kind = "reference" if O.have_reference() else "port"
    rows = 96
    band = full[p.ny // 2:p.ny // 2 + rows].cpu().numpy()
    pb = abi.make_problem(2, p.nx, rows, p.dx, p.dy, a_g=p.a_g, cfl=p.cfl)
    t0 = time.perf_counter()
    ref = R.snapshot_to_string(pb, band, 12.5)
    cpu_s = time.perf_counter() - t0
    mine = native.snapshot_to_string(pb, band, 12.5)
    out = {"workload": a.workload, "cells": cells, "bytes": nbytes, "sink": a.sink,
           "gpu_seconds": gpu_s, "gpu_cells_per_s": cells / gpu_s,
           "gpu_GB_per_s": nbytes / gpu_s / 1e9,
           "cpu_kind": kind, "cpu_cells": p.nx * rows, "cpu_seconds": cpu_s,
           "cpu_cells_per_s": p.nx * rows / cpu_s, "sample_identical": mine == ref}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
