"""Expected outcomes of the reference's physics acceptance criteria, computed
by the REFERENCE itself (oracle/_ref/libsilt_ref.so, its own scenario
builders and run_serial):

  1  periodic dune conserves water and bed  (proj/tests/acceptance_main.cpp:104-126)
  2  dam break = plain shallow water         (:130-160)
  3  dune migration + refinement             (:164-195)
  4  antidune upstream migration             (:199-225)
  9  lake at rest: spurious |u| shrinks      (:395-415)
  10 planar bump crescent                    (:419-449)

    make -C oracle && python tests/golden/make_golden_acceptance.py   (~10 min)
    python tests/golden/make_golden_acceptance.py --extra   (criteria 1, 2, 9 only; merged)

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


def conservation_case(R):
    """Criterion 1's scenario: dune1d(500) between periodic ends, 1000 steps."""
    from paper_1307_0491_b200 import abi
    p, init, _ = R.build_scenario("dune1d", 500)
    p.bc[abi.WEST] = abi.bc("periodic")
    p.bc[abi.EAST] = abi.bc("periodic")
    return p, init


def volumes(f, dx):
    """water_volume / bed_volume (acceptance_main.cpp:49-59), summed in cell order."""
    w = b = 0.0
    for c in f.reshape(-1, 4):
        w += float(c[0])
        b += float(c[3])
    return w * dx, b * dx


def dam_break_case():
    """Criterion 2's scenario: 400 cells on [0, 200] m, h = 2 | 1 at x = 100,
    no transport (Grass A_g = 0), t_end = 10 s, transmissive ends."""
    from paper_1307_0491_b200 import abi
    n = 400
    p = abi.make_problem(1, n, 1, 200.0 / n, 1.0, a_g=0.0, cfl=0.5)
    f = np.zeros((1, n, 4))
    x = (np.arange(n) + 0.5) * (200.0 / n)
    f[0, :, 0] = np.where(x < 100.0, 2.0, 1.0)
    return p, f, 10.0


def lake_case(R, cells):
    """Criterion 9's scenario: dune1d(cells) with Grass A_g = 0, walls, hu = 0, t_end = 20."""
    from paper_1307_0491_b200 import abi
    p, init, _ = R.build_scenario("dune1d", cells)
    p.a_g = 0.0
    p.bc[abi.WEST] = abi.bc("wall")
    p.bc[abi.EAST] = abi.bc("wall")
    init = init.copy()
    init[..., 1] = 0.0
    return p, init, 20.0


def umax(f):
    return float(np.max(np.abs(f[..., 1] / f[..., 0])))


def extra(R):
    """Criteria 1, 2, 9 on the reference (run_serial through oracle/_ref)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import kats
    out = {}
    p, init = conservation_case(R)
    f, t, steps, _ = R.run(p, init, t_end=1e6, max_steps=1000)
    w0, b0 = volumes(init, p.dx)
    w1, b1 = volumes(f, p.dx)
    out["conservation"] = {"steps": steps, "water_drift": abs(w1 - w0) / w0,
                           "bed_drift": abs(b1 - b0) / b0}
    p, f0, t_end = dam_break_case()
    f, t, steps, _ = R.run(p, f0, t_end=t_end)
    rh, rhu = kats.suliciu_run(f0[0, :, 0], f0[0, :, 1], p.dx, t_end)
    gap = max(float(np.max(np.abs(f[0, :, 0] - rh))), float(np.max(np.abs(f[0, :, 1] - rhu))))
    out["dam_break"] = {"t": t, "steps": steps, "gap": gap,
                        "bed_clean": bool(np.all(f[..., 3] == 0.0))}
    lake = {}
    for cells in (500, 1000):
        p, init, t_end = lake_case(R, cells)
        f, t, steps, _ = R.run(p, init, t_end=t_end)
        lake[str(cells)] = {"umax": umax(f), "steps": steps, "t": t}
    out["lake"] = lake
    return out


def main():
    import oracle as O
    R = O.reference()
    if "--extra" in sys.argv:
        path = os.path.join(HERE, "golden_acceptance.json")
        with open(path) as fh:
            out = json.load(fh)
        out.update(extra(R))
        print({k: out[k] for k in ("conservation", "dam_break", "lake")}, flush=True)
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
        return

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
    out.update(extra(R))
    with open(os.path.join(HERE, "golden_acceptance.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
