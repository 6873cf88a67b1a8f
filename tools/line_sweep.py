"""Per-step time of 1D lines of increasing length (C1 physics), one solver,
n steps per call: python tools/line_sweep.py [steps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1307_0491_b200 import native, scenarios
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
for nx in (360, 720, 1000, 1440, 2000, 2880, 4000, 5760):
    p, init, _ = scenarios.dune_1d(nx)
    s = native.Solver(p)
    s.upload(init)
    s.begin(max_steps=steps + 10)
    s.step(10); s.status()
    t0 = time.perf_counter()
    s.step(steps); s.status()
    el = time.perf_counter() - t0
    print(f"nx {nx:5d} ctas {(nx + 359) // 360:2d}: {el / steps * 1e6:.2f} us/step", flush=True)
    s.close()
