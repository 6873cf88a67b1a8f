import sys, time, os
sys.path.insert(0,'.')
import numpy as np
from paper_1307_0491_b200 import native, scenarios, abi
for name, build, steps in (("C1", scenarios.dune_1d, 1000), ("C2", scenarios.antidune_1d, 5000), ("C3", lambda: scenarios.dune_2d(1024), 1000)):
    p, init, _ = build()
    s = native.Solver(p)
    s.upload(init)
    s.begin(max_steps=steps + 10)
    s.step(10); s.status()
    t0 = time.perf_counter()
    s.step(steps); st = s.status()
    el = time.perf_counter() - t0
    print(name, steps, f"{el*1e3:.2f} ms total, {el/steps*1e6:.2f} us/step, {p.nx*p.ny*steps/el/1e9:.3f} G cell/s", flush=True)
    s.close()
