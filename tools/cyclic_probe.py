#!/usr/bin/env python
"""Per-GPU step time of a CYCLIC row distribution, emulated on one GPU.

    python tools/cyclic_probe.py [--workload C4] [--n 8] [--blocks 4]

GPU g of n owns row blocks g, g+n, g+2n, ... (n * blocks blocks of equal
height); each block is its own solver on its own stream (neighbour rows
frozen), all launched concurrently, so the CTAs of the blocks mix on the SMs
like one launch.  Prints, for every g, the time of one such step (CUDA events
around the concurrent launches), and the contiguous-strip time for comparison.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1307_0491_b200 import abi, native  # noqa: E402
from paper_1307_0491_b200.distributed import _CAI  # noqa: E402


def make(p, full, j0, n):
    strip = abi.SiltStrip(j0, n, 1 if j0 > 0 else 0, 1 if j0 + n < p.ny else 0)
    s = native.Solver(p, strip, 0, abi.VARIANT_FAST)
    st = torch.cuda.Stream()
    s.set_stream(st.cuda_stream)
    rows = full[j0:j0 + n].contiguous()
    torch.cuda.synchronize()
    s.upload_device(rows.data_ptr())
    ex = s.exchange_ptrs()
    for ptr, row in ((ex.recv_south, j0 - 1), (ex.recv_north, j0 + n)):
        if ptr:
            t = torch.as_tensor(_CAI(ptr, 4 * p.nx), device="cuda")
            t.copy_(full[row].t().contiguous().reshape(-1))
    torch.cuda.synchronize()
    return s, st


def timed(solvers, steps, warmup):
    for s, _ in solvers:
        s.begin(max_steps=steps + warmup + 1)
    base = torch.cuda.current_stream()
    for s, _ in solvers:
        s.step(warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(base)
    for s, st in solvers:
        st.wait_stream(base)
    for k in range(steps):  # interleave the blocks' launches step by step
        for s, _ in solvers:
            s.step(1)
    for s, st in solvers:
        base.wait_stream(st)
    e1.record(base)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--blocks", type=int, default=4)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    p = bench.build_global_problem(a.workload, 1)
    full = bench.device_initial_rows(a.workload, p, 0, p.ny, torch.device("cuda"))
    nblk = a.n * a.blocks
    h = p.ny // nblk
    worst = 0.0
    for g in range(a.n):
        solvers = [make(p, full, (g + a.n * k) * h, h) for k in range(a.blocks)]
        ms = timed(solvers, a.steps, 3)
        worst = max(worst, ms)
        print(f"gpu {g}: {a.blocks} blocks of {h} rows  {ms:.3f} ms/step", flush=True)
        for s, _ in solvers:
            s.close()
    print(f"cyclic max {worst:.3f} ms/step")


if __name__ == "__main__":
    main()
