"""Two pieces per rank, concurrently (strong scaling on C4).

Rank r of N owns 1/N of the hot band around the mound (rows [0.38, 0.62] of
the grid: the mound and the waves it sends out) and 1/N of the far field (the
lower far-field range for the first N/2 ranks, the upper one for the rest).
Both pieces step as two solvers on two streams of the same GPU, so the hot
piece's FP64-bound CTAs overlap with the far field's HBM-bound ones — as in
the one-GPU launch — and the hot piece uses short row blocks (SILT_ROWS) so
that its CTAs are not a tail.  Each piece's ghost rows stay frozen at the
initial neighbour rows (as in tools/strip_times.py).  Prints the per-rank
step time (max over ranks) and efficiency = T1 / (N * max).

    python tools/two_piece_probe.py [--ns 4,8] [--hot-rows 8,16,24]
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
from paper_1307_0491_b200 import abi, native  # noqa: E402
from paper_1307_0491_b200.distributed import _CAI, block_range  # noqa: E402
from strip_times import strip_ms  # noqa: E402


def make_solver(p, full, j0, n, rows_env):
    if rows_env:
        os.environ["SILT_ROWS"] = str(rows_env)
    else:
        os.environ.pop("SILT_ROWS", None)
    strip = abi.SiltStrip(j0, n, 1 if j0 > 0 else 0, 1 if j0 + n < p.ny else 0)
    s = native.Solver(p, strip, 0, abi.VARIANT_FAST)
    os.environ.pop("SILT_ROWS", None)
    stream = torch.cuda.Stream()
    s.set_stream(stream.cuda_stream)
    rows = full[j0:j0 + n].contiguous()
    torch.cuda.synchronize()
    s.upload_device(rows.data_ptr())
    ex = s.exchange_ptrs()
    for ptr, row in ((ex.recv_south, j0 - 1), (ex.recv_north, j0 + n)):
        if ptr:
            t = torch.as_tensor(_CAI(ptr, 4 * p.nx), device="cuda")
            t.copy_(full[row].t().contiguous().reshape(-1))
    return s, stream, rows


def rank_ms(p, full, pieces, steps, warmup):
    """Step both pieces concurrently (one stream each); ms per step."""
    ss = [make_solver(p, full, j0, n, rr) for j0, n, rr in pieces]
    for s, _, _ in ss:
        s.begin(max_steps=steps + warmup + 1)
    for _ in range(warmup):
        for s, _, _ in ss:
            s.step(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    e0.record(main)
    for _, st, _ in ss:
        st.wait_stream(main)
    for _ in range(steps):
        for s, _, _ in ss:
            s.step(1)
    for _, st, _ in ss:
        main.wait_stream(st)
    e1.record(main)
    torch.cuda.synchronize()
    for s, _, _ in ss:
        s.close()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--ns", default="4,8")
    ap.add_argument("--hot-rows", default="8,16,24")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    p = bench.build_global_problem(a.workload, 1)
    full = bench.device_initial_rows(a.workload, p, 0, p.ny, torch.device("cuda"))
    t1 = strip_ms(p, full, 0, p.ny, a.steps, a.warmup)
    lo, hi = int(0.38 * p.ny), int(0.62 * p.ny)
    print(f"T1 {t1:.3f} ms; hot band rows [{lo}, {hi})", flush=True)
    for n in map(int, a.ns.split(",")):
        half = n // 2
        for hr in [int(x) for x in a.hot_rows.split(",")]:
            ts = []
            for r in range(n):
                h0, hc = block_range(hi - lo, n, r)
                if r < half:
                    f0, fc = block_range(lo, half, r)
                else:
                    f0, fc = block_range(p.ny - hi, n - half, r - half)
                    f0 += hi
                pieces = [(lo + h0, hc, hr), (f0, fc, 0)]
                ts.append(rank_ms(p, full, pieces, a.steps, a.warmup))
            eff = t1 / (n * max(ts))
            print(f"N={n} hot rows/block {hr}: max {max(ts):.3f} ms, efficiency {eff:.2f}; ranks "
                  + " ".join(f"{x:.3f}" for x in ts), flush=True)


if __name__ == "__main__":
    main()
