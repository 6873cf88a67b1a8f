"""Per-CTA timeline of one 2D step launch (needs a -DSILT_TRACE build):
SILT_LIB=exp/trace/libsilt_b200.so python tools/cta_trace.py C4 300 [out.npz]
Runs `steps` steps, traces the next one, and prints where the launch's time
goes: hot (full-path) vs quiescent CTAs, occupancy over time, the tail."""
import ctypes as C, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_1307_0491_b200 import native

wl, steps = sys.argv[1], int(sys.argv[2])
out = sys.argv[3] if len(sys.argv) > 3 else None
p = bench.build_global_problem(wl, 1)
init = bench.device_initial_rows(wl, p, 0, p.ny, torch.device("cuda"))
torch.cuda.synchronize()
L = native.lib()
s = native.Solver(p)
s.upload_device(init.data_ptr())
s.begin(max_steps=steps + 2)
if steps:
    s.step(steps)
s.status()
nrec = 1 << 22
buf = torch.zeros(nrec, 4, dtype=torch.int64, device="cuda")
buf[:, 0] = -1
L.silt_debug_trace(C.c_void_p(buf.data_ptr()))
s.step(1)
s.status()
L.silt_debug_trace(C.c_void_p(0))
r = buf.cpu().numpy().view(np.uint64)
r = r[r[:, 1] > 0]
t0 = r[:, 0].min()
st = (r[:, 0] - t0) / 1e3
en = (r[:, 1] - t0) / 1e3
sm = (r[:, 2] & 0xFFFF).astype(int)
rb = (r[:, 3] & 0xFFFFFFFF).astype(int)
full = (r[:, 3] >> 32).astype(int)
dur = en - st
T = en.max()
hot = full > 0
print(f"{wl} step {steps + 1}: {len(r)} CTAs, launch {T:.1f} us")
for name, m in (("hot (any full-path row)", hot), ("quiescent", ~hot)):
    if m.any():
        print(f"  {name}: {m.sum()} CTAs, duration mean {dur[m].mean():.1f} us, "
              f"p50 {np.median(dur[m]):.1f}, p99 {np.percentile(dur[m], 99):.1f}, max {dur[m].max():.1f}; "
              f"sum {dur[m].sum() / 1e3:.1f} CTA-ms; last end {en[m].max():.1f} us")
q = np.sort(en)
for f in (0.5, 0.9, 0.95, 0.99, 1.0):
    print(f"  {int(f * 100)}% of CTAs done at {q[min(len(q) - 1, int(f * len(q)))]:.1f} us")
# resident CTAs (all / hot) over time, in 20 bins
edges = np.linspace(0, T, 21)
mid = 0.5 * (edges[1:] + edges[:-1])
res = [((st <= x) & (en > x)).sum() for x in mid]
resh = [((st <= x) & (en > x) & hot).sum() for x in mid]
print("  resident CTAs over time (all / hot):")
print("   " + " ".join(f"{a}/{b}" for a, b in zip(res, resh)))
# hot CTAs started late
late = hot & (st > 0.8 * T)
print(f"  hot CTAs started after 80% of the launch: {late.sum()}, their last end {en[late].max() if late.any() else 0:.1f} us")
if out:
    np.savez_compressed(out, st=st, en=en, sm=sm, rb=rb, full=full)
