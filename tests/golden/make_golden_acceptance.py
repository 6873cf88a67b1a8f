"""Expected outcomes of the reference's physics acceptance criteria, computed
by the REFERENCE itself (oracle/_ref/libsilt_ref.so, its own scenario
builders and run_serial):

  3  dune migration + refinement  (proj/tests/acceptance_main.cpp:164-195)
  4  antidune upstream migration  (:199-225)
  10 planar bump crescent         (:419-449)

    make -C oracle && python tests/golden/make_golden_acceptance.py   (~10 min)

tests/test_acceptance.py runs the same scenarios on the GPU path and compares
the crest tracks, bed L1 gaps, inflow Froude numbers and bed maxima with
these values (and the criteria's verdicts with the reference's).
"""
from __future__ import annotations

import json
import math
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

DUNE_SNAPS = [100.0 * k for k in range(8)]          # acceptance_main.cpp:167
ANTIDUNE_SNAPS = [0.0, 6.0, 10.0, 15.0, 30.0, 50.0]  # :203


def crest_track(snaps, dx):
    """crest_track (src/report.cpp:74-110): x of the highest bed cell per
    snapshot (ties -> smallest x) and the monotonicity verdict."""
    xs = []
    for f in snaps:
        zb = f[..., 3]
        best = None
        for j in range(zb.shape[0]):
            i = int(np.argmax(zb[j]))  # first maximum of the row: the smallest x
            if best is None or zb[j, i] > best[0] or (zb[j, i] == best[0] and i < best[1]):
                best = (zb[j, i], i)
        xs.append((best[1] + 0.5) * dx)
    up = any(b < a for a, b in zip(xs, xs[1:]))
    down = any(b > a for a, b in zip(xs, xs[1:]))
    verdict = "mixed" if up and down else "downstream" if down else "upstream" if up \
        else "stationary"
    return xs, verdict


def coarsen2(f):
    """acceptance_main.cpp:62-71 (1D)."""
    a, b = f[0, 0::2], f[0, 1::2]
    out = np.zeros((1, a.shape[0], 4))
    out[0, :, 0] = 0.5 * (a[:, 0] + b[:, 0])
    out[0, :, 1] = 0.5 * (a[:, 1] + b[:, 1])
    out[0, :, 3] = 0.5 * (a[:, 3] + b[:, 3])
    return out


def l1_bed_diff(a, b, dx):
    """acceptance_main.cpp:73-78."""
    s = 0.0
    for x, y in zip(a[0, :, 3], b[0, :, 3]):
        s += abs(x - y)
    return s * dx


def bump_split(field):
    """split_max of check_bump_shape (acceptance_main.cpp:425-437)."""
    ny = field.shape[0]
    zb = field[..., 3]
    centre_rows = [ny // 2 - 1, ny // 2]
    centre = max(zb[j].max() for j in centre_rows)
    off = max(zb[j].max() for j in range(ny) if j not in centre_rows)
    return float(centre), float(off)


def main():
    import oracle as O
    R = O.reference()

    def dune(cells):
        p, init, t_end = R.build_scenario("dune1d", cells)
        snaps = DUNE_SNAPS if cells == 2000 else [t_end]
        fields, t, steps = R.run_snaps(p, init, t_end, snaps)
        return cells, p.dx, fields, steps

    with ThreadPoolExecutor(3) as ex:
        runs = {c: r for c, *r in ex.map(dune, [2000, 4000, 8000])}
    dx2000, snaps, steps2000 = runs[2000]
    xs, verdict = crest_track(snaps, dx2000)
    f2000, f4000, f8000 = snaps[-1], runs[4000][1][-1], runs[8000][1][-1]
    d_coarse = l1_bed_diff(f2000, coarsen2(f4000), dx2000)
    d_fine = l1_bed_diff(f4000, coarsen2(f8000), runs[4000][0])
    out = {"generator": "tests/golden/make_golden_acceptance.py",
           "source": "oracle/_ref/libsilt_ref.so (reference core) run_serial + its scenario builders",
           "dune": {"snapshots": DUNE_SNAPS, "crest_x": xs, "verdict": verdict,
                    "l1_coarse": d_coarse, "l1_fine": d_fine,
                    "steps": {str(c): runs[c][2] for c in (2000, 4000, 8000)}}}
    print("dune", out["dune"], flush=True)

    p, init, _ = R.build_scenario("antidune1d", 2400)
    fields, t, steps = R.run_snaps(p, init, 50.0, ANTIDUNE_SNAPS)
    xs, verdict = crest_track(fields, p.dx)
    fr = [float((f[0, 0, 1] / f[0, 0, 0]) / math.sqrt(p.gravity * f[0, 0, 0])) for f in fields]
    out["antidune"] = {"snapshots": ANTIDUNE_SNAPS, "crest_x": xs, "verdict": verdict,
                       "inflow_froude": fr, "steps": steps}
    print("antidune", out["antidune"], flush=True)

    p, init, t_end = R.build_scenario("bump2d", 200, 200, 1.0)
    fields, t, steps = R.run_snaps(p, init, t_end, [t_end])
    c0, o0 = bump_split(init)
    c1, o1 = bump_split(fields[-1])
    out["bump"] = {"t_end": t_end, "steps": steps, "centre0": c0, "off0": o0, "centre1": c1,
                   "off1": o1, "lowered": c1 < c0, "split": o1 > c1}
    print("bump", out["bump"], flush=True)
    with open(os.path.join(HERE, "golden_acceptance.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
