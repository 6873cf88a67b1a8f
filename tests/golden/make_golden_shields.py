"""Generate the Shields-law golden fixtures from the REFERENCE itself.

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden_shields.py

Every array comes from oracle/_ref/libsilt_ref.so (the unmodified reference
core, oracle/ref_driver.cpp) for BedloadLaw::shields with each of the five
ShieldsFormula values and both FrictionModel values
(include/silt/bedload.hpp:12-52):
  * law probes  — dimensional_flux, dqs_du, normal_flux, normal_flux_derivative,
                  shields_stress, friction_slope on seeded (h, u_n, u_t) states;
  * formula probes — shields_flux / shields_flux_derivative on a tau grid;
  * interface solves — solve_face (src/stepper.cpp:69-89) on seeded cell pairs;
  * whole runs — run_serial (src/parallel.cpp:208-259), 2D and 1D.
Written to golden_shields.npz / golden_shields.json next to this script.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)

import oracle as O  # noqa: E402
from make_golden import face_pairs  # noqa: E402
from paper_1307_0491_b200 import abi, scenarios as S  # noqa: E402

FORMULAS = list(abi.SHIELDS_FORMULAS)
FRICTIONS = list(abi.FRICTION_MODELS)


def law_states(seed: int, n: int) -> np.ndarray:
    """(h, u_n, u_t) covering dry, at rest, below / near / above threshold."""
    rng = np.random.default_rng(seed)
    X = np.empty((n, 3))
    X[:, 0] = rng.uniform(0.05, 12.0, n)
    X[:, 1] = rng.uniform(-4.0, 4.0, n)
    X[:, 2] = rng.uniform(-2.0, 2.0, n)
    m = n // 8
    X[:m, 2] = 0.0                      # aligned flow
    X[m:m + 4, 1:] = 0.0                # at rest
    X[m + 4:m + 8, 0] = 0.0             # dry
    X[m + 8:m + 12, 1] = 5e-11          # below kUEps
    X[m + 8:m + 12, 2] = 0.0
    X[m + 12:2 * m, 1:] *= 0.05         # slow: mostly below threshold
    return X


def shields_problem(formula: str, friction: str, **kw):
    p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=0.0)
    return abi.set_shields(p, formula, friction, **kw)


def law_meta(p) -> dict:
    return {"formula": FORMULAS[p.shields_formula], "friction": FRICTIONS[p.friction_model],
            "friction_coef": p.friction_coef, "tau_cr": p.tau_cr,
            "grain_diameter": p.grain_diameter, "rel_density": p.rel_density}


def main() -> None:
    R = O.reference()
    meta: dict = {"generator": "tests/golden/make_golden_shields.py",
                  "source": "oracle/_ref/libsilt_ref.so (reference core, -O3 -DNDEBUG)",
                  "cases": {}}
    arrays: dict = {}

    # ---- formula probes: q*(tau), dq*/dtau --------------------------------------
    tau = np.concatenate([[0.0, 1e-12, 0.02, 0.047, 0.05, 0.0470000001],
                          np.linspace(0.0, 3.0, 61), np.geomspace(1e-6, 50.0, 40)])
    arrays["formula_tau"] = tau
    for k, f in enumerate(FORMULAS):
        for tc in (0.047, 0.0):
            arrays[f"formula_{f}_tc{tc}"] = R.shields_flux(k, tau, tc)

    # ---- law probes and interface solves per (formula, friction) -----------------
    X = law_states(1307, 512)
    arrays["law_states"] = X
    for i, f in enumerate(FORMULAS):
        for j, fr in enumerate(FRICTIONS):
            p = shields_problem(f, fr)
            tag = f"{f}_{fr}"
            arrays[f"law_{tag}"] = R.law_eval(p, X)
            Lc, Rc = face_pairs(900 + 10 * i + j, 256)
            arrays[f"faces_{tag}_L"] = Lc
            arrays[f"faces_{tag}_R"] = Rc
            for axis in (0, 1):
                arrays[f"faces_{tag}_ax{axis}_out"] = R.faces(p, Lc, Rc, axis)[0]
            meta["cases"][f"law_{tag}"] = law_meta(p)

    # ---- whole runs ---------------------------------------------------------------
    def run_case(tag, p, init, steps, bcs=None, snaps=()):
        if bcs is not None:
            for s in range(4):
                p.bc[s] = bcs[s]
        out, t, n, log = R.run(p, init, max_steps=steps, snapshots=snaps)
        arrays[f"{tag}_init"] = init
        arrays[f"{tag}_final"] = out
        arrays[f"{tag}_dt"] = log
        meta["cases"][tag] = {
            "dim": p.dim, "nx": p.nx, "ny": p.ny, "dx": p.dx, "dy": p.dy,
            "a_g": p.a_g, "m_g": p.m_g, "cfl": p.cfl, "safety": p.safety,
            "law": law_meta(p),
            "bc": [[p.bc[s].type, p.bc[s].supercritical, p.bc[s].q0, p.bc[s].h0]
                   for s in range(4)],
            "max_steps": steps, "t_end": None, "snapshots": list(snaps),
            "steps": n, "t_final": t,
            "bed_moved": float(np.abs(out[..., 3] - init[..., 3]).max())}
        print(tag, n, repr(t), meta["cases"][tag]["bed_moved"], flush=True)

    for f in FORMULAS:
        for fr in FRICTIONS:
            p, init, _ = S.random_bed_2d(24, 16, a_g=0.0)
            abi.set_shields(p, f, fr)
            run_case(f"run2d_{f}_{fr}", p, init, 25)
    p, init, _ = S.dune_1d(cells=128)
    abi.set_shields(p, "mpm", "manning")
    run_case("run1d_mpm_manning", p, init, 60)
    p, init, _ = S.dune_1d(cells=128)
    abi.set_shields(p, "camenen", "darcy-weisbach")
    run_case("run1d_camenen_darcy-weisbach", p, init, 60)
    p, init, _ = S.dune_2d(48, a_g=0.0)
    abi.set_shields(p, "nielsen", "darcy-weisbach", tau_cr=0.2)
    run_case("dune48_nielsen_dw_tc0.2", p, init, 40,
             bcs=[abi.bc("inflow", q0=10.0), abi.bc("outflow"), abi.bc("wall"), abi.bc("wall")],
             snaps=(0.5,))
    # coarse grain: tau << tau_cr everywhere, the bed must not move at all
    p, init, _ = S.dune_2d(32, a_g=0.0)
    abi.set_shields(p, "mpm", "manning", grain_diameter=0.2)
    run_case("frozen_coarse_mpm", p, init, 30)

    np.savez_compressed(os.path.join(HERE, "golden_shields.npz"), **arrays)
    with open(os.path.join(HERE, "golden_shields.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
