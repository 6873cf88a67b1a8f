"""Newton statistics of the FAST fluid-outer solver (needs a -DSILT_STATS build:
SILT_LIB=exp/stats/libsilt_b200.so python tools/newton_stats.py C5 10)."""
import ctypes as C, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_1307_0491_b200 import native
wl, steps = sys.argv[1], int(sys.argv[2])
p = bench.build_global_problem(wl, 1)
init = bench.device_initial_rows(wl, p, 0, p.ny, torch.device("cuda"))
torch.cuda.synchronize()
L = native.lib()
st = (C.c_ulonglong * 8)()
s = native.Solver(p)
s.upload_device(init.data_ptr())
s.begin(max_steps=steps + 1)
s.step(1); s.status(); L.silt_debug_stats(st, 8)
for k in range(steps):
    s.step(1); s.status()
    L.silt_debug_stats(st, 8)
    n, it, zero, early = st[0], st[1], st[2], st[3]
    print(f"{wl} step {k+1}: fluid-outer solves {n}, Newton its/solve {it/max(n,1):.3f}, "
          f"at-guess {zero/max(n,1):.3f}, early-accept {early/max(n,1):.3f}")
