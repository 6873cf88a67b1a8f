"""Generate the large-grid fixtures (C3, C4, C5) from the REFERENCE itself.

Run in the build container (where /root/reference exists; ~30 min on 8 cores):
    make -C oracle && python tests/golden/make_golden_big.py [C3 C4w C5]

The fields are too large to commit, so each case stores, per row and per field,
a 64-bit BLAKE2b digest of the reference's final field (the row's nx doubles,
little-endian) plus the full dt log and t_final.  A row digest match is a
bit-for-bit match of that row, so the STRICT GPU run is compared with the
reference on EVERY cell; the FAST run is then compared with the STRICT run on
the full field (tests/test_gpu_big.py).  Digests of the initial fields are kept
too, so a test fails loudly if a host builds different inputs.

Every field comes from oracle/_ref/libsilt_ref.so (the unmodified reference
core) through ref_run_blocks: run_parallel's loop on row strips through the
public API (partition / halo_exchange / apply_bc_side / cfl_dt / global_dt /
step_2d), bitwise equal to run_serial (the reference's layout contract,
tests/test_parallel.cpp:215-238; checked on small grids in tests/test_oracle.py).

Cases
  C3   BASELINE configs[2]: 1024^2 dune, A_g = 0.001, CFL 0.5, 1000 steps, whole grid.
  C4w  BASELINE configs[3] (16384^2 dune, 500 steps) on the window
       [lo - m, hi + m)^2 around the mound's non-uniform cells with m = 508.
       Outside the mound the initial state is bitwise uniform (h = 9.9, hu = 10,
       hv = 0, zb = 0.1), a uniform state is a fixed point of the step, and a
       disturbance spreads at most one cell per step, so for k < m - 1 steps the
       window with transmissive sides evolves bit for bit like the same cells
       of the full 16384^2 grid, with the same dt (the window holds far-field
       cells, so the maxima of the axis speeds and of h agree).  The full grid
       outside the window stays exactly uniform.
  C5   BASELINE configs[4]'s generator (scenarios.random_bed_2d) on the per-GPU
       tile 8192 x 4096 (bench.py --workload C5 at N = 1), A_g = 0.01, CFL 0.4,
       100 steps: every face takes the full solver.
  C4w40_fma / C4w500_fma / C3_fma
       The reference's own rounding spread: the same reference sources compiled
       with FMA contraction (oracle/_ref/libsilt_ref_fma.so, `make -C oracle
       ref_fma`) against the default build, per field (normwise), on the C4
       window after 40 and 500 steps and on C3 after 1000 steps.  Early in the C4 run hv
       is O(1e-7) while the y-momentum fluxes it is the difference of are
       O(500), so its per-field ratio there measures rounding: the reference
       disagrees with itself by ~1e-5 (tests/test_gpu_parity.py uses this as
       the hv bar of its 40-step C4 property test).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_1307_0491_b200 import scenarios as S  # noqa: E402

C4_MARGIN = 508
C4_STEPS = 500
C5_STEPS = 100


def row_digests(field: np.ndarray) -> np.ndarray:
    """(ny, 4) uint64: BLAKE2b-64 of each row of each field of an AoS field."""
    ny = field.shape[0]
    out = np.empty((ny, 4), dtype=np.uint64)
    for f in range(4):
        plane = np.ascontiguousarray(field[:, :, f])
        for j in range(ny):
            out[j, f] = np.frombuffer(hashlib.blake2b(plane[j].tobytes(), digest_size=8).digest(),
                                      dtype="<u8")[0]
    return out


def field_digest(field: np.ndarray) -> str:
    return hashlib.blake2b(np.ascontiguousarray(field).tobytes(), digest_size=16).hexdigest()


def c4_window(n: int = 16384, margin: int = C4_MARGIN):
    """[lo, hi) of the window per axis (x: columns, y: rows)."""
    dx = 1000.0 / n
    wx = S._sine_bump(S._centres(n, dx), 300.0, 200.0)
    wy = S._sine_bump(S._centres(n, dx), 400.0, 200.0)
    nzx = np.nonzero(wx)[0]
    nzy = np.nonzero(wy)[0]
    return ((int(nzx[0]) - margin, int(nzx[-1]) + 1 + margin),
            (int(nzy[0]) - margin, int(nzy[-1]) + 1 + margin))


def c4_window_problem(margin: int = C4_MARGIN):
    """The C4 problem restricted to the window: same dx/dy, outflow sides."""
    n = 16384
    (x0, x1), (y0, y1) = c4_window(n, margin)
    p_full, _, _ = S.dune_2d(64)  # law/cfl of C3/C4; grid replaced below
    from paper_1307_0491_b200 import abi
    dx = 1000.0 / n
    p = abi.make_problem(2, x1 - x0, y1 - y0, dx, dx, a_g=p_full.a_g, cfl=p_full.cfl)
    wx = S._sine_bump(S._centres(n, dx), 300.0, 200.0)[x0:x1]
    wy = S._sine_bump(S._centres(n, dx), 400.0, 200.0)[y0:y1]
    init = np.zeros((y1 - y0, x1 - x0, 4))
    zb = 0.1 + np.multiply.outer(wy, wx)
    init[..., 0] = 10.0 - zb
    init[..., 1] = 10.0
    init[..., 3] = zb
    return p, init, ((x0, x1), (y0, y1))


def fma_spread(name: str, threads: int):
    """Per-field normwise difference between the FMA-contracted reference
    build and the default build (both the unmodified reference sources)."""
    import oracle as O
    R = O.reference()
    F = O.CpuSolver(os.path.join(ROOT, "oracle", "_ref", "libsilt_ref_fma.so"), "ref")
    if name == "C4w40_fma":
        p, init, win = c4_window_problem(48)
        steps, py = 40, 64
    elif name == "C4w500_fma":
        p, init, win = c4_window_problem()
        steps, py = C4_STEPS, 128
    else:
        p, init, steps = S.dune_2d(1024, steps=1000)
        py = 64
    a = R.run_blocks(p, init, steps, py, threads)
    b = F.run_blocks(p, init, steps, py, threads)
    A, B = a[0].reshape(-1, 4), b[0].reshape(-1, 4)
    meta = {"steps": steps, "nx": p.nx, "ny": p.ny,
            "max_abs": np.abs(A).max(0).tolist(),
            "fma_vs_ref_normwise": (np.abs(A - B).max(0) / np.abs(A).max(0)).tolist(),
            "fma_vs_ref_dt": float(np.max(np.abs(a[3] - b[3]) / a[3]))}
    print(name, meta, flush=True)
    return meta, {}


def run_case(name: str, threads: int):
    import oracle as O
    if name.endswith("_fma"):
        return fma_spread(name, threads)
    R = O.reference()
    meta: dict = {}
    if name == "C3":
        p, init, steps = S.dune_2d(1024, steps=1000)
        py = 64
    elif name == "C4w":
        p, init, win = c4_window_problem()
        steps = C4_STEPS
        py = 128
        meta["window"] = {"x": list(win[0]), "y": list(win[1]), "margin": C4_MARGIN,
                          "n": 16384}
    elif name == "C5":
        p, init, _ = S.random_bed_2d(8192, 4096)
        steps = C5_STEPS
        py = 128
    else:
        raise SystemExit(f"unknown case {name}")
    t0 = time.time()
    out, t, n, log = R.run_blocks(p, init, steps, py, threads)
    el = time.time() - t0
    assert n == steps
    meta.update({"nx": p.nx, "ny": p.ny, "dx": p.dx, "dy": p.dy, "a_g": p.a_g, "cfl": p.cfl,
                 "steps": n, "t_final": t, "init_digest": field_digest(init),
                 "final_digest": field_digest(out), "ref_seconds": el, "threads": threads,
                 "strips": py})
    arrays = {f"{name}_rows": row_digests(out), f"{name}_dt": log,
              f"{name}_init_rows": row_digests(init)}
    print(f"{name}: {p.nx}x{p.ny} x {n} steps in {el:.0f} s, t_final {t!r}", flush=True)
    return meta, arrays


def main(argv):
    cases = argv or ["C3", "C4w", "C5"]
    threads = os.cpu_count() or 1
    path_j = os.path.join(HERE, "golden_big.json")
    path_z = os.path.join(HERE, "golden_big.npz")
    meta = {"generator": "tests/golden/make_golden_big.py",
            "source": "oracle/_ref/libsilt_ref.so (reference core, -O3 -DNDEBUG) via ref_run_blocks",
            "digest": "blake2b digest_size=8 per row per field (little-endian uint64)",
            "cases": {}}
    arrays: dict = {}
    if os.path.exists(path_j):
        with open(path_j) as fh:
            meta["cases"] = json.load(fh)["cases"]
        old = np.load(path_z)
        arrays = {k: old[k] for k in old.files}
    for c in cases:
        m, a = run_case(c, threads)
        meta["cases"][c] = m
        arrays.update(a)
        with open(path_j, "w") as fh:
            json.dump(meta, fh, indent=1)
        np.savez_compressed(path_z, **arrays)


if __name__ == "__main__":
    main(sys.argv[1:])
