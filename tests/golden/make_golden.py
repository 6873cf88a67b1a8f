"""Generate the committed golden fixtures from the REFERENCE itself.

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py

Every array is produced by oracle/_ref/libsilt_ref.so — the unmodified
reference core compiled from /root/reference/proj/core/src — through its public
API (oracle/ref_driver.cpp).  The fixtures let the CPU test-suite pin the C
restatement and the GPU parity tests run without the reference tree.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_1307_0491_b200 import abi, scenarios as S  # noqa: E402


def face_pairs(seed: int, n: int):
    """Random cell pairs covering wet/dry, sub/supercritical, flat/stepped bed."""
    rng = np.random.default_rng(seed)
    L = np.empty((n, 4))
    R = np.empty((n, 4))
    for k, side in ((0, L), (1, R)):
        h = rng.uniform(0.3, 4.0, n)
        side[:, 0] = h
        side[:, 1] = h * rng.uniform(-4.0, 4.0, n)
        side[:, 2] = h * rng.uniform(-1.0, 1.0, n)
        side[:, 3] = rng.uniform(-0.5, 0.5, n)
    # structured sub-populations
    m = n // 8
    R[:m] = L[:m]                                   # uniform data (invisible fan)
    R[m:2 * m, 3] = L[m:2 * m, 3]                   # flat bed
    L[2 * m:3 * m, 1] = 0.0                         # at rest on one side
    L[2 * m:3 * m, 2] = 0.0
    L[3 * m:3 * m + 8, 0] = 0.0                     # dry left
    L[3 * m + 8:3 * m + 16, 0] = 0.5e-8             # below h_dry with stale discharge
    R[3 * m + 16:3 * m + 24, 0] = 0.0               # dry right
    L[3 * m + 24:3 * m + 28] = 0.0                  # both dry
    R[3 * m + 24:3 * m + 28] = 0.0
    return L, R


def main() -> None:
    R = O.reference()
    meta: dict = {"generator": "tests/golden/make_golden.py",
                  "source": "oracle/_ref/libsilt_ref.so (reference core, -O3 -DNDEBUG)",
                  "cases": {}}
    arrays: dict = {}

    # ---- interface solves (solve_face, src/stepper.cpp:69-89) ------------------
    for tag, a_g, seed in (("faces_ag0p3", 0.3, 503), ("faces_ag0p001", 0.001, 504),
                           ("faces_ag0", 0.0, 505), ("faces_ag5", 5.0, 506)):
        p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=a_g)
        Lc, Rc = face_pairs(seed, 512)
        for axis in (0, 1):
            out, info = R.faces(p, Lc, Rc, axis)
            arrays[f"{tag}_ax{axis}_L"] = Lc
            arrays[f"{tag}_ax{axis}_R"] = Rc
            arrays[f"{tag}_ax{axis}_out"] = out
            arrays[f"{tag}_ax{axis}_info"] = info
        meta["cases"][tag] = {"a_g": a_g, "seed": seed, "n": 512}

    # ---- whole runs --------------------------------------------------------------
    def run_case(tag, p, init, steps, snaps=(), t_end=np.inf, bcs=None):
        if bcs is not None:
            for s in range(4):
                p.bc[s] = bcs[s]
        t0 = time.time()
        out, t, n, log = R.run(p, init, max_steps=steps, t_end=t_end, snapshots=snaps)
        arrays[f"{tag}_init"] = init
        arrays[f"{tag}_final"] = out
        arrays[f"{tag}_dt"] = log
        meta["cases"][tag] = {
            "dim": p.dim, "nx": p.nx, "ny": p.ny, "dx": p.dx, "dy": p.dy,
            "a_g": p.a_g, "m_g": p.m_g, "cfl": p.cfl, "safety": p.safety,
            "bc": [[p.bc[s].type, p.bc[s].supercritical, p.bc[s].q0, p.bc[s].h0]
                   for s in range(4)],
            "max_steps": steps, "t_end": None if np.isinf(t_end) else t_end,
            "snapshots": list(snaps), "steps": n, "t_final": t,
            "seconds": round(time.time() - t0, 2)}
        print(tag, n, repr(t), f"{time.time() - t0:.1f}s", flush=True)

    p, init, steps = S.dune_1d()
    run_case("C1", p, init, steps)
    p, init, steps = S.antidune_1d()
    run_case("C2", p, init, steps)
    p, init, _ = S.random_bed_2d(48, 32, steps=60)
    run_case("rand48x32", p, init, 60)
    p, init, _ = S.dune_2d(64, a_g=1.0)
    run_case("dune64_ag1", p, init, 80)
    p, init, _ = S.random_bed_2d(40, 24, a_g=0.3)
    run_case("bc_inflow_wall", p, init, 40, snaps=(0.5, 1.0),
             bcs=[abi.bc("inflow", q0=1.0), abi.bc("outflow"), abi.bc("wall"), abi.bc("outflow")])
    p, init, _ = S.random_bed_2d(40, 24, a_g=0.3)
    run_case("bc_periodic", p, init, 40, bcs=[abi.bc("periodic")] * 4)
    p, init, _ = S.random_bed_2d(40, 24, a_g=0.3)
    run_case("bc_supercrit_tend", p, init, 1000, t_end=1.5,
             bcs=[abi.bc("inflow", q0=1.0, h0=0.2, supercritical=True), abi.bc("wall"),
                  abi.bc("periodic"), abi.bc("periodic")])
    p, init, _ = S.dune_1d(cells=64)
    run_case("periodic_ring1d", p, init, 200, bcs=[abi.bc("periodic"), abi.bc("periodic"),
                                                 abi.bc("outflow"), abi.bc("outflow")])

    # ---- C3 at full size: row checksums only (32 MiB field is not committed) ------
    p, init, steps = S.dune_2d(1024, steps=1000)
    t0 = time.time()
    threads = os.cpu_count() or 1
    out, t, n, comp, wall = R.run_parallel(p, init, 1, threads, max_steps=steps)
    arrays["C3_rowsum"] = out.sum(axis=1)          # (1024, 4) per-row sums
    arrays["C3_colsum"] = out.sum(axis=0)          # (1024, 4) per-column sums
    arrays["C3_probe"] = out[::97, ::89].copy()    # sparse probe of cells
    # dt log for the first 20 steps (serial loop)
    _, _, _, log20 = R.run(p, init, max_steps=20)
    arrays["C3_dt20"] = log20
    meta["cases"]["C3"] = {"nx": 1024, "ny": 1024, "steps": n, "t_final": t,
                           "threads": threads, "seconds": round(time.time() - t0, 1),
                           "sum_h": float(out[..., 0].sum()), "sum_hu": float(out[..., 1].sum()),
                           "sum_zb": float(out[..., 3].sum())}
    print("C3", n, repr(t), f"{time.time() - t0:.1f}s")

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
