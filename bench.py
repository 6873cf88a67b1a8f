#!/usr/bin/env python
"""Benchmark of the B200-native relaxation time step (arXiv 1307.0491).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4|C3|C5]
                    [--impl ours|reference] [--variant fast|strict]

Metric (BASELINE.json): fp64 2D cell-updates/s, whole job, with the fraction
of the HBM roofline.  A "step" is one time step of the fused kernel over the
whole grid (all strips).  Default workload C4 = the 16384^2 dune of
BASELINE.json configs[3] (the north star's strong-scaling grid; 8.6 GB of
state per copy, far larger than L2, so no L2 flush is needed).  N > 1 runs
under torchrun: one process per GPU, row strips, NCCL halo rows + MAX
all-reduce of the CFL speeds (paper_1307_0491_b200.distributed).

`--impl reference` times the reference's own CPU implementation
(oracle/_ref, the unmodified reference core) on this host's cores over a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_CELL = 64  # h, hu, hv, zb fp64 read once + written once
FALLBACK_HBM_GBS = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


WORKLOADS = {
    # name: (builder kwargs, description)
    "C3": dict(kind="dune", n=1024, a_g=0.001, cfl=0.5),
    "C4": dict(kind="dune", n=16384, a_g=0.001, cfl=0.5),
    "C4s": dict(kind="dune", n=4096, a_g=0.001, cfl=0.5),  # profiling size
    "C5": dict(kind="random", nx=8192, ny_per_gpu=4096, a_g=0.01, cfl=0.4),
    "Q": dict(kind="uniform", n=16384, a_g=0.001, cfl=0.5),  # diagnostics: quiescent-row path
}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.samples)}


def apply_law(p, law: str):
    """--law grass (BASELINE's workloads) or <formula>:<friction>, e.g.
    mpm:manning — BedloadLaw::shields with the config layer's defaults."""
    from paper_1307_0491_b200 import abi
    if law != "grass":
        formula, friction = law.split(":")
        abi.set_shields(p, formula, friction)
    return p


def build_global_problem(wl: str, world: int, law: str = "grass"):
    from paper_1307_0491_b200 import abi
    w = WORKLOADS[wl]
    if w["kind"] in ("dune", "uniform"):
        n = w["n"]
        p = abi.make_problem(2, n, n, 1000.0 / n, 1000.0 / n, a_g=w["a_g"], cfl=w["cfl"])
    else:
        ny = w["ny_per_gpu"] * world
        p = abi.make_problem(2, w["nx"], ny, 1.0, 1.0, a_g=w["a_g"], cfl=w["cfl"])
    return apply_law(p, law)


def device_initial_rows(wl: str, p, j0: int, nrows: int, device):
    """Initial AoS rows [j0, j0+nrows) built on the device (bitwise equal to
    scenarios.dune_2d / the reference's sine_bump construction)."""
    import numpy as np
    import torch
    from paper_1307_0491_b200 import scenarios as S
    w = WORKLOADS[wl]
    nx = p.nx
    out = torch.zeros((nrows, nx, 4), dtype=torch.float64, device=device)
    if w["kind"] == "uniform":
        out[..., 0] = 9.9
        out[..., 1] = 10.0
        out[..., 3] = 0.1
    elif w["kind"] == "dune":
        wx = torch.from_numpy(S._sine_bump(S._centres(nx, p.dx), 300.0, 200.0)).to(device)
        wy_all = S._sine_bump(S._centres(p.ny, p.dy), 400.0, 200.0)
        wy = torch.from_numpy(np.ascontiguousarray(wy_all[j0:j0 + nrows])).to(device)
        zb = 0.1 + torch.outer(wy, wx)
        out[..., 0] = 10.0 - zb
        out[..., 1] = 10.0
        out[..., 3] = zb
    else:
        # C5: the seeded 8192 x 4096 tile (scenarios.random_bed_2d; periodic
        # Gaussian random field) repeated along y, so the global field is the
        # same for every GPU count and N = 1 is exactly the reference-pinned
        # tile (tests/test_gpu_big.py)
        tile = c5_tile(nx)
        rows = (np.arange(j0, j0 + nrows) % tile.shape[0])
        out.copy_(torch.from_numpy(np.ascontiguousarray(tile[rows])))
    return out


_TILES: dict = {}


def c5_tile(nx: int):
    """The C5 random-bed tile (nx x ny_per_gpu, BASELINE configs[4] per GPU)."""
    from paper_1307_0491_b200 import scenarios as S
    if nx not in _TILES:
        w = WORKLOADS["C5"]
        _, _TILES[nx], _ = S.random_bed_2d(nx, w["ny_per_gpu"], a_g=w["a_g"], cfl=w["cfl"])
    return _TILES[nx]


def cpu_model() -> str:
    """Host CPU model (for the CPU-baseline report)."""
    name, fam, model = "unknown", "?", "?"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                k, _, v = line.partition(":")
                k, v = k.strip(), v.strip()
                if k == "model name" and name == "unknown":
                    name = v
                elif k == "cpu family" and fam == "?":
                    fam = v
                elif k == "model" and model == "?":
                    model = v
    except OSError:
        pass
    return f"{name} (family {fam} model {model}), {os.cpu_count()} logical CPUs"


def host_workload(wl: str, world: int, law: str = "grass"):
    """(problem, AoS initial field) of the whole workload on the host — the
    same grid, law and initial data our arm uploads (bitwise: the device
    builder of device_initial_rows restates these constructions)."""
    from paper_1307_0491_b200 import scenarios as S
    w = WORKLOADS[wl]
    p = build_global_problem(wl, world, law)
    if w["kind"] == "dune":
        _, init, _ = S.dune_2d(w["n"])
    elif w["kind"] == "uniform":
        import numpy as np
        init = np.zeros((p.ny, p.nx, 4))
        init[..., 0] = 9.9
        init[..., 1] = 10.0
        init[..., 3] = 0.1
    else:
        import numpy as np
        tile = c5_tile(w["nx"])
        init = np.ascontiguousarray(tile[np.arange(p.ny) % tile.shape[0]])
    return p, init


def cpu_reference_window(wl: str, world: int, steps_lo: int, steps_hi: int, threads: int,
                         law: str = "grass"):
    """The reference's own CPU driver, silt::run_parallel(sc, 1, P) (oracle/_ref,
    the unmodified reference core), on the WHOLE workload grid: cell-updates/s
    over steps [steps_lo, steps_hi) from t = 0, timed by the reference's own
    WorkerTiming.compute_seconds (src/parallel.cpp:318-361; max over workers):
    one run of steps_hi steps minus one of steps_lo steps."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    p, init = host_workload(wl, world, law)
    if O.have_reference():
        R, kind = O.reference(), "reference"
    else:  # the GPU box always has the prebuilt oracle/_ref; the port is the fallback
        R, kind, threads = O.restatement(), "port", 1
    P = max(1, min(threads, p.ny))

    def compute(n):
        if n <= 0:
            return 0.0, 0
        if kind == "reference":
            _, _, ns, comp, _ = R.run_parallel(p, init, 1, P, max_steps=n, want_field=False)
            return comp, ns
        t0 = time.perf_counter()
        _, _, ns, _ = R.run(p, init, max_steps=n, dt_log=False)
        return time.perf_counter() - t0, ns

    c_lo, n_lo = compute(steps_lo)
    c_hi, n_hi = compute(steps_hi)
    assert n_hi - n_lo == steps_hi - steps_lo
    rate = p.nx * p.ny * (n_hi - n_lo) / (c_hi - c_lo)
    desc = (f"{wl} whole grid {p.nx}x{p.ny}, steps [{steps_lo}, {steps_hi}) from t=0, "
            f"run_parallel(sc, 1, {P}), WorkerTiming.compute_seconds")
    return rate, desc, kind, P


def cpu_reference_band_p1(wl: str, law: str = "grass"):
    """Single-thread reference rate, run_parallel(sc, 1, 1), on a 96-row band of
    the workload (the whole grid at P = 1 would take minutes per step)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.have_reference():
        return None
    from paper_1307_0491_b200 import abi
    p_full, init_full = host_workload(wl, 1, law) if WORKLOADS[wl].get("n", 0) <= 4096 \
        else (None, None)
    w = WORKLOADS[wl]
    if p_full is None:  # a C4-sized dune: build only the band
        from paper_1307_0491_b200 import scenarios as S
        n = w["n"]
        rows = 96
        j0 = int(0.45 * n)
        dx = 1000.0 / n
        wx = S._sine_bump(S._centres(n, dx), 300.0, 200.0)
        wy = S._sine_bump(S._centres(n, dx), 400.0, 200.0)[j0:j0 + rows]
        init = np.zeros((rows, n, 4))
        zb = 0.1 + np.multiply.outer(wy, wx)
        init[..., 0] = 10.0 - zb
        init[..., 1] = 10.0
        init[..., 3] = zb
        p = abi.make_problem(2, n, rows, dx, dx, a_g=w["a_g"], cfl=w["cfl"])
        apply_law(p, law)
        desc = f"rows [{j0},{j0 + rows}) x {n}, 1 step"
    else:
        rows = min(96, p_full.ny)
        init = np.ascontiguousarray(init_full[:rows])
        p = abi.make_problem(2, p_full.nx, rows, p_full.dx, p_full.dy, a_g=p_full.a_g,
                             cfl=p_full.cfl)
        apply_law(p, law)
        desc = f"rows [0,{rows}) x {p.nx}, 1 step"
    _, _, ns, comp, _ = O.reference().run_parallel(p, init, 1, 1, max_steps=1, want_field=False)
    return {"value": p.nx * p.ny * ns / comp, "unit": "cell-updates/s", "cores": 1,
            "sample": desc}


def workload_config(args, p) -> dict:
    """The workload both arms run (identical dicts: the driver compares them)."""
    return {"workload": f"{args.workload} ({p.nx}x{p.ny}, A_g={p.a_g}, CFL={p.cfl})",
            "law": args.law, "nx": p.nx, "ny": p.ny}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    lo, hi = args.warmup, args.warmup + args.steps
    value, desc, kind, used = cpu_reference_window(args.workload, args.gpus, lo, hi, threads,
                                                   args.law)
    p = build_global_problem(args.workload, args.gpus, args.law)
    line = {
        "metric": "cell-updates/s (fp64, 2D)", "value": value, "unit": "cell-updates/s",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "weak" if WORKLOADS[args.workload]["kind"] == "random" else "strong",
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, p),
        "reference_run": {"driver": f"silt::run_parallel(sc, 1, {used}) (oracle/_ref)",
                          "timing": f"compute_seconds(run of {hi} steps) - compute_seconds(run "
                                    f"of {lo} steps): the {args.steps} steps after {lo} "
                                    "warm-up steps",
                          "cpu": cpu_model(), "threads": used},
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": used, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # 500: BASELINE's C4 strong-scaling run
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="fast", choices=["fast", "strict"])
    ap.add_argument("--law", default="grass",
                    help="grass (BASELINE workloads) or <formula>:<friction>, "
                         "formula in mpm|flvb|nielsen|ribberink|camenen, "
                         "friction in manning|darcy-weisbach")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--partition", default="balanced", choices=["balanced", "uniform"],
                    help="row strips for N > 1: equal estimated work (default) or block_range")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    from paper_1307_0491_b200 import abi, native
    from paper_1307_0491_b200.distributed import (PieceRunner, StripRunner, balanced_partition,
                                                  init_dist, piece_partition, refine_partition,
                                                  row_costs)

    world, rank, local = init_dist(args.gpus)
    # one GPU per rank; ranks beyond the visible devices share them (only for
    # the one-GPU multi-rank check with SILT_DIST_BACKEND=gloo)
    local = local % max(1, torch.cuda.device_count())
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    variant = abi.VARIANT_FAST if args.variant == "fast" else abi.VARIANT_STRICT
    p = build_global_problem(args.workload, world, args.law)
    partition = None
    layout = None  # two pieces per rank (PieceRunner)
    if world > 1 and args.partition == "balanced" and WORKLOADS[args.workload]["kind"] == "dune":
        # Work-balanced layouts (quiescent rows are cheaper).  Every rank
        # derives the same cut from the same initial field.  Default: two
        # pieces per rank (1/N of the hot band around the mound + 1/N of the
        # far field, stepped concurrently: DESIGN.md §6); SILT_PIECES=0 (or no
        # peer memory) keeps contiguous strips, whose cut a short untimed
        # pilot rescales by each strip's measured step time.
        full = device_initial_rows(args.workload, p, 0, p.ny, device)
        costs = row_costs(full)
        del full
        torch.cuda.empty_cache()
        # pieces from N = 4 (tools/strip_times.py --pieces, C4: N = 2 pieces 0.88 vs
        # strips 0.98, N = 4 0.88 vs 0.83, N = 8 0.87 vs 0.78); SILT_PIECES_MIN overrides
        min_n = int(os.environ.get("SILT_PIECES_MIN", "4"))
        if (world >= min_n and os.environ.get("SILT_PIECES", "1") != "0"
                and os.environ.get("SILT_P2P", "1") != "0"):
            layout = piece_partition(costs, world)
        partition = balanced_partition(costs, world)
        for _ in range(0 if layout else 2):  # two measured refinements
            pilot = StripRunner(p, world, rank, device=local, variant=variant,
                                partition=partition)
            pilot.upload_device(device_initial_rows(args.workload, p, pilot.j0, pilot.nrows,
                                                    device))
            pilot.begin(max_steps=8)
            pilot.step(3)
            pilot.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(pilot.torch_stream)
            pilot.solver.step(4)  # this strip alone (its step kernels)
            e1.record(pilot.torch_stream)
            torch.cuda.synchronize()
            mine = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
            times = [torch.zeros_like(mine) for _ in range(world)]
            torch.distributed.all_gather(times, mine)
            pilot.close()
            partition = refine_partition(costs, partition, [float(x.item()) for x in times])
            torch.cuda.empty_cache()
    if layout:
        try:
            runner = PieceRunner(p, world, rank, layout, device=local, variant=variant)
        except RuntimeError:  # no peer memory between the ranks: contiguous strips (NCCL)
            layout = None
    if layout:
        runner.upload_rows(lambda a, n: device_initial_rows(args.workload, p, a, n, device))
        j0, nrows = runner.j0, runner.nrows
    else:
        runner = StripRunner(p, world, rank, device=local, variant=variant, partition=partition)
        j0, nrows = runner.j0, runner.nrows
        init = device_initial_rows(args.workload, p, j0, nrows, device)
        runner.upload_device(init)
        del init
    total = args.warmup + args.steps
    runner.begin(max_steps=total + 1)
    runner.step(args.warmup)
    runner.synchronize()

    stream = runner.torch_stream
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    n0 = runner.launch_count()
    runner.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        runner.record_join()
        ev0.record(stream)
        runner.step(args.steps)
        runner.record_join()
        ev1.record(stream)
        torch.cuda.synchronize()
    runner.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = runner.launch_count() - n0
    ms = runner.max_over_ranks(ms)
    st = runner.status()
    assert st.steps == total, (st.steps, total)

    cells = p.nx * p.ny
    value = cells * args.steps / (ms / 1e3)
    ms_step = ms / args.steps
    peak, peak_src = peaks()
    # per-GPU average (strips may be uneven: work-balanced partition); the
    # step time is the max over ranks
    per_gpu_cells = cells / world
    achieved = per_gpu_cells * BYTES_PER_CELL / (ms_step / 1e3) / 1e9
    traffic = None
    fp64_roof = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tj = json.load(fh)
        tr = tj.get(args.workload)
        if tr:
            traffic = tr["dram_bytes_per_launch"] * (per_gpu_cells / tr["cells"])
        # Active flow is bound by the FP64 pipe, not HBM: FP64-pipe thread
        # instructions per cell-update (DFMA+DMUL+DADD+DSETP, from the committed
        # ncu capture of this workload) x cell-updates/s, against the measured
        # DFMA rate (profiles/r1_fp64_peak.json; one FP64-pipe instruction each).
        with open(os.path.join(ROOT, "profiles", "r1_fp64_peak.json")) as fh:
            fp_peak = float(json.load(fh)["dfma_per_s"])
        if tr and tr.get("fp64_pipe_inst_per_cell") and args.variant == "fast":
            per_cell = tr["fp64_pipe_inst_per_cell"]
            ach = per_gpu_cells / (ms_step / 1e3) * per_cell
            fp64_roof = {"bound": "fp64", "achieved": ach / 1e12, "peak": fp_peak / 1e12,
                         "unit": "T FP64-pipe thread instr/s", "frac": ach / fp_peak,
                         "per_cell": per_cell,
                         "source": "profiles/" + tr.get("source", "?") + " opcode mix ("
                                   + tr.get("capture", "one step launch") + "); peak "
                                   "profiles/r1_fp64_peak.json"}
    except Exception:
        pass

    # end to end through the public API (silt_run semantics): pinned host
    # field -> device, K steps, device -> pinned host
    e2e = None
    if not args.no_e2e:
        ranges = ([(q["j0"], q["n"]) for q in runner.pieces] if layout else [(j0, nrows)])
        hosts = []
        for a, n in ranges:
            h = torch.empty((n, p.nx, 4), dtype=torch.float64, pin_memory=True)
            h.copy_(device_initial_rows(args.workload, p, a, n, device).cpu())
            hosts.append(h)
        outs = [torch.empty_like(h, pin_memory=True) for h in hosts]
        if layout:
            runner2 = PieceRunner(p, world, rank, layout, device=local, variant=variant)
        else:
            runner2 = StripRunner(p, world, rank, device=local, variant=variant,
                                  partition=partition)
        runner2.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if layout:
            runner2.upload_host_tensors(hosts)
        else:
            runner2.upload_host(hosts[0])
        runner2.begin(max_steps=args.steps)
        runner2.step(args.steps)
        if layout:
            runner2.download_host_tensors(outs)
        else:
            runner2.download_host(outs[0])
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        runner2.barrier()
        el = runner.max_over_ranks(el)
        nbytes = sum(h.numel() for h in hosts) * 8 * world
        e2e = {"value": cells * args.steps / el, "unit": "cell-updates/s",
               "h2d_bytes_per_step": int(nbytes / args.steps),
               "d2h_bytes_per_step": int(nbytes / args.steps),
               "timing": "wall clock around upload+begin+K steps+download, max over ranks"}
        runner2.close()
        del hosts, outs

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rate, desc, kind, used = cpu_reference_window(args.workload, 1, 0, 2,
                                                          os.cpu_count() or 1, args.law)
            cpu = {"value": rate, "unit": "cell-updates/s", "cores": used, "kind": kind,
                   "sample": desc, "cpu": cpu_model()}
            if args.workload in ("C3", "C4", "C4s"):
                cpu["p1"] = cpu_reference_band_p1(args.workload, args.law)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "cell-updates/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "cell-updates/s (fp64, 2D)",
            "value": value,
            "unit": "cell-updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak" if WORKLOADS[args.workload]["kind"] == "random" else "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "variant": args.variant,
            "config": workload_config(args, p),
            "layout": {"rows_per_gpu": nrows, "parallelism": f"row strips x{world}",
                       "partition": ("two pieces per rank: " + str(layout) if layout
                                     else args.partition if world > 1 else "single strip"),
                       "l2": ("state 64 B/cell x %d cells >> 126 MB L2; no flush" % cells
                              if 64 * cells > 4 * 126e6 else
                              "state 64 B/cell x %d cells is L2-sized; not flushed (a step re-reads "
                              "the previous step's output: L2-resident by design)" % cells)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src,
                         "note": "algorithmic 64 B/cell-update / device time per step (the step "
                                 "kernel plus, in launches >= 64 CTAs/SM, the 1-CTA "
                                 "rb_order_kernel that orders the next launch, ~0.1 %)"},
            "roofline_fp64": fp64_roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    runner.close()
    runner.shutdown()
    return 0


if __name__ == "__main__":
    sys.exit(main())
