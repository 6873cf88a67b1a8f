#!/usr/bin/env python
"""Per-strip step time of a row partition, measured strip by strip on ONE GPU.

    python tools/strip_times.py [--workload C4] [--steps 20] [--warmup 5]

For N = 2, 4, 8 and the uniform (block_range) and work-balanced partitions,
each strip is run as its own solver (its ghost rows stay frozen at the
initial neighbour rows) and its step kernel is timed with CUDA events.  The
max over strips estimates the N-GPU compute time per step (communication not
included); efficiency = T1 / (N * max_k T_k).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1307_0491_b200 import abi, native  # noqa: E402
from paper_1307_0491_b200.distributed import (balanced_partition, block_range,  # noqa: E402
                                              refine_partition, row_costs)


def strip_ms(p, full, j0, n, steps, warmup):
    strip = abi.SiltStrip(j0, n, 1 if j0 > 0 else 0, 1 if j0 + n < p.ny else 0)
    s = native.Solver(p, strip, 0, abi.VARIANT_FAST)
    stream = torch.cuda.Stream()
    s.set_stream(stream.cuda_stream)
    strip_rows = full[j0:j0 + n].contiguous()
    torch.cuda.synchronize()  # order torch's producer before the solver's copy
    s.upload_device(strip_rows.data_ptr())
    ex = s.exchange_ptrs()
    for ptr, row in ((ex.recv_south, j0 - 1), (ex.recv_north, j0 + n)):
        if ptr:  # freeze the neighbour rows at their initial values
            t = torch.as_tensor(__import__("paper_1307_0491_b200.distributed",
                                           fromlist=["_CAI"])._CAI(ptr, 4 * p.nx), device="cuda")
            t.copy_(full[row].t().contiguous().reshape(-1))
    s.begin(max_steps=steps + warmup + 1)
    s.step(warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.step(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    s.close()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ns", default="2,4,8", help="strip counts to measure")
    ap.add_argument("--pieces", action="store_true",
                    help="also the two-pieces-per-rank layout (distributed.piece_partition)")
    a = ap.parse_args()
    p = bench.build_global_problem(a.workload, 1)
    full = bench.device_initial_rows(a.workload, p, 0, p.ny, torch.device("cuda"))
    costs = row_costs(full)
    t1 = strip_ms(p, full, 0, p.ny, a.steps, a.warmup)
    out = {"workload": a.workload, "t1_ms": t1, "runs": []}
    for n in [int(x) for x in a.ns.split(",")]:
        bal = balanced_partition(costs, n)
        bal_t = [strip_ms(p, full, j0, c, 4, 3) for j0, c in bal]  # pilot 1
        ref1 = refine_partition(costs, bal, bal_t)
        ref1_t = [strip_ms(p, full, j0, c, 4, 3) for j0, c in ref1]  # pilot 2
        for name, part in (("uniform", [block_range(p.ny, n, r) for r in range(n)]),
                           ("balanced", bal),
                           ("refined", refine_partition(costs, ref1, ref1_t))):
            ts = [strip_ms(p, full, j0, c, a.steps, a.warmup) for j0, c in part]
            eff = t1 / (n * max(ts))
            out["runs"].append({"n": n, "partition": name, "rows": [c for _, c in part],
                                "strip_ms": ts, "max_ms": max(ts), "efficiency": eff})
            print(f"N={n} {name:8s} max {max(ts):.3f} ms  eff {eff:.2f}  strips "
                  + " ".join(f"{x:.2f}" for x in ts), flush=True)
        if a.pieces:
            from two_piece_probe import rank_ms
            from paper_1307_0491_b200.distributed import piece_partition
            layout = piece_partition(costs, n)
            hr = int(os.environ.get("SILT_PIECE_HOT_ROWS", "32"))
            ts = [rank_ms(p, full, [(h0, hn, hr), (f0, fn, 0)], a.steps, a.warmup)
                  for (h0, hn), (f0, fn) in layout]
            eff = t1 / (n * max(ts))
            out["runs"].append({"n": n, "partition": "pieces", "layout": layout, "rank_ms": ts,
                                "max_ms": max(ts), "efficiency": eff})
            print(f"N={n} pieces   max {max(ts):.3f} ms  eff {eff:.2f}  ranks "
                  + " ".join(f"{x:.2f}" for x in ts), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
