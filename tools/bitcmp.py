#!/usr/bin/env python
"""A/B numerics of two library builds: run the same workloads through each
(SILT_LIB picks the build, one subprocess per build) and compare the final
fields bitwise (and normwise per field when they differ) plus the dt logs.

    python tools/bitcmp.py LIB_A LIB_B [--steps 200]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = {
    # name: (builder, kwargs, steps)
    "c3": ("dune_2d", dict(n=1024), 300),
    "c5s": ("random_bed_2d", dict(nx=1024, ny=512), 200),
    "c5b": ("random_bed_2d", dict(nx=2048, ny=1024, seed=7), 100),
}


def _child(out_dir: str, steps_scale: float):
    sys.path.insert(0, ROOT)
    from paper_1307_0491_b200 import native, scenarios as S
    for name, (fn, kw, steps) in CASES.items():
        p, init, _ = getattr(S, fn)(**kw)
        n = max(1, int(steps * steps_scale))
        out, t, k, log = native.run(p, init, max_steps=n)
        np.savez(os.path.join(out_dir, name + ".npz"), out=out, log=log, t=t, k=k)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib_a")
    ap.add_argument("lib_b")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--child", default=None)
    a = ap.parse_args()
    if a.child:
        _child(a.child, a.scale)
        return
    dirs = []
    for lib in (a.lib_a, a.lib_b):
        d = tempfile.mkdtemp()
        env = dict(os.environ, SILT_LIB=os.path.abspath(lib))
        subprocess.run([sys.executable, __file__, lib, lib, "--child", d, "--scale", str(a.scale)],
                       env=env, check=True)
        dirs.append(d)
    worst = 0.0
    for name in CASES:
        x = np.load(os.path.join(dirs[0], name + ".npz"))
        y = np.load(os.path.join(dirs[1], name + ".npz"))
        same = np.array_equal(x["out"].view(np.int64), y["out"].view(np.int64))
        errs = []
        for f in range(4):
            xa, ya = x["out"][..., f], y["out"][..., f]
            den = max(np.abs(xa).max(), 1e-300)
            errs.append(float(np.abs(xa - ya).max() / den))
        worst = max(worst, max(errs))
        dtd = float(np.abs(x["log"] - y["log"]).max() / np.abs(x["log"]).max()) if len(x["log"]) else 0
        print(f"{name}: steps {int(x['k'])}/{int(y['k'])} bitwise={same} "
              f"field err {['%.2e' % e for e in errs]} dt err {dtd:.2e}")
    print(f"worst normwise field difference {worst:.3e}")


if __name__ == "__main__":
    main()
