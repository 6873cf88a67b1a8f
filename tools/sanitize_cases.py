"""Small runs of every device path under the bounds-CHECKED library build.

compute-sanitizer is closed on this GPU pool (it answers "runs under it have
left GPUs needing a reset", profiles/r2_sanitizer.md), so the kernels carry
their own checks: build them with

    python -m paper_1307_0491_b200.build --out paper_1307_0491_b200/lib/checked/libsilt_b200.so \
        --extra -DSILT_CHECKED
    SILT_LIB=paper_1307_0491_b200/lib/checked/libsilt_b200.so python tools/sanitize_cases.py

Every global row / column index, ring slot and DSMEM slot is validated before
the access (violations counted and skipped, silt_debug_checks).  Each case is
also compared with the C restatement (oracle/, test infrastructure): STRICT
bitwise, FAST within 1e-9 normwise.  No torch: only our kernels run.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_1307_0491_b200 import abi, native  # noqa: E402
from paper_1307_0491_b200.distributed import LocalStripGroup  # noqa: E402


def field(nx, ny, seed):
    rng = np.random.default_rng(seed)
    f = np.empty((ny, nx, 4))
    f[..., 3] = 0.1 + 0.05 * rng.random((ny, nx))
    f[..., 0] = 1.5 - f[..., 3] + 0.05 * rng.random((ny, nx))
    f[..., 1] = f[..., 0] * rng.uniform(0.2, 0.8, (ny, nx))
    f[..., 2] = f[..., 0] * rng.uniform(-0.2, 0.2, (ny, nx)) if ny > 1 else 0.0
    return f


def normwise(a, b):
    a = a.reshape(-1, 4)
    b = b.reshape(-1, 4)
    den = np.maximum(np.abs(b).max(0), 1e-300)
    return (np.abs(a - b).max(0) / den).max()


CHECKED = [None]


def violations():
    import ctypes as C
    L = native.lib()
    out = (C.c_ulonglong * 4)()
    CHECKED[0] = bool(L.silt_debug_checks(out))
    return list(out)


def check(name, got, ref, strict):
    ok = np.array_equal(got, ref) if strict else normwise(got, ref) <= 1e-9
    v = violations()
    print(f"{name}: {'ok' if ok else 'MISMATCH'}; bounds violations {v[0]}"
          + (f" (first: code {v[1]}, {v[2]}, {v[3]})" if v[0] else ""), flush=True)
    if not ok or v[0]:
        raise SystemExit(1)


def main():
    orc = O.restatement()
    bcsets = {
        "outflow": [abi.bc("outflow")] * 4,
        "inflow/wall/periodic": [abi.bc("inflow", q0=0.7), abi.bc("wall"), abi.bc("periodic"),
                                 abi.bc("periodic")],
        "periodic/wall/outflow": [abi.bc("periodic"), abi.bc("periodic"), abi.bc("wall"),
                                  abi.bc("outflow")],
        "supercritical inflow": [abi.bc("inflow", q0=2.0, h0=0.3, supercritical=True),
                                 abi.bc("outflow"), abi.bc("wall"), abi.bc("wall")],
    }
    # 2D step kernel, both variants, every BC type, a width that is no
    # multiple of the 30-column warp band
    init = field(67, 45, 1)
    for label, bcs in bcsets.items():
        p = abi.make_problem(2, 67, 45, 1.0, 1.0, a_g=0.3, bcs=bcs)
        ref = orc.run(p, init, max_steps=8)[0]
        for vname, v in (("strict", abi.VARIANT_STRICT), ("fast", abi.VARIANT_FAST)):
            got = native.run(p, init, max_steps=8, variant=v)[0]
            check(f"2d {label} {vname}", got, ref, v == abi.VARIANT_STRICT)
    # quiescent rows (FAST skip + streak loop): uniform flow around a bump
    u = np.zeros((70, 95, 4))
    u[..., 3] = 0.1
    u[30:34, 40:44, 3] = 0.3
    u[..., 0] = 2.0 - u[..., 3]
    u[..., 1] = 1.2
    p = abi.make_problem(2, 95, 70, 1.0, 1.0, a_g=0.01, cfl=0.45)
    ref = orc.run(p, u, max_steps=6)[0]
    check("2d quiescent fast", native.run(p, u, max_steps=6, variant=abi.VARIANT_FAST)[0], ref,
          False)
    # repeated rows (STRICT skip + streak loop), long row blocks
    os.environ["SILT_ROWS"] = "40"
    check("2d repeated rows strict", native.run(p, u, max_steps=6, variant=abi.VARIANT_STRICT)[0],
          ref, True)
    # warp items through the row-block order table (forced on a small grid)
    os.environ.update(SILT_ROWS="8", SILT_ROW_PERM="1", SILT_WARP_ITEMS="1")
    for vname, v in (("strict", abi.VARIANT_STRICT), ("fast", abi.VARIANT_FAST)):
        check(f"2d ordered warp items {vname}", native.run(p, u, max_steps=6, variant=v)[0], ref,
              v == abi.VARIANT_STRICT)
    for k in ("SILT_ROWS", "SILT_ROW_PERM", "SILT_WARP_ITEMS"):
        os.environ.pop(k)
    # 1D: single launches, resident cluster (<= 8 CTAs), global-memory cluster,
    # cooperative grid
    for nx in (37, 2000, 4000, 6100):
        line = field(nx, 1, nx)
        p = abi.make_problem(1, nx, 1, 1.0, 1.0, a_g=0.3)
        ref = orc.run(p, line, max_steps=12)[0]
        for vname, v in (("strict", abi.VARIANT_STRICT), ("fast", abi.VARIANT_FAST)):
            got = native.run(p, line, max_steps=12, variant=v)[0]
            check(f"1d nx={nx} {vname}", got, ref, v == abi.VARIANT_STRICT)
    # strip group, direct mode (edge rows stored into the neighbours' receive
    # rows, maxima by remote atomics), 3 strips on one device
    init = field(64, 60, 3)
    p = abi.make_problem(2, 64, 60, 1.0, 1.0, a_g=0.3)
    ref = orc.run(p, init, max_steps=10)[0]
    g = LocalStripGroup(p, 3, devices=(0,), variant=abi.VARIANT_STRICT)
    g.upload(init)
    g.begin(max_steps=10)
    g.run(batch=4)
    check("strip group x3 strict", g.gather(), ref, True)
    g.close()
    # snapshots: pause on the device clock, asynchronous capture
    s = native.Solver(p, variant=abi.VARIANT_STRICT)
    s.upload(init)
    s.begin(max_steps=40, snapshots=[0.5, 1.0])
    seen = []
    s.run(batch=3, on_snapshot=lambda t, f: seen.append(t), async_snapshots=True)
    s.close()
    v = violations()
    print("snapshots landed:", seen, "; bounds violations", v[0], flush=True)
    if v[0] or seen != [0.5, 1.0]:
        raise SystemExit(1)
    print(f"sanitize cases done (checked build: {CHECKED[0]})", flush=True)


if __name__ == "__main__":
    main()
