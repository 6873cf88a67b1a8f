"""CPU stand-in for one CUDA strip solver — TEST INFRASTRUCTURE ONLY.

Implements the strip-solver interface that paper_1307_0491_b200.distributed.
StripRunner drives (begin / step / status / resume / download / reduce slot /
exchange buffers) with the oracle restatement doing the per-strip step, so the
multi-rank host logic (partition, neighbour order, periodic wrap, MAX
all-reduce of the axis speeds, snapshot pauses, gather) can be tested with the
gloo backend on CPU.  It mirrors the device protocol of the CUDA strip:
  * begin: reduce state 0 into the slot, write edge rows to send buffers;
  * step:  dt = cfl * min(dx / max_sx, dy / max_sy) from the (all-reduced)
           slot, clipped like run_serial; ghosts = physical BCs or received
           rows; step_2d on the padded strip; reduce the new state.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from paper_1307_0491_b200 import abi


class StripStatus:
    def __init__(self, t, steps, state, snap):
        self.t, self.steps, self.state, self.snapshot_index = t, steps, state, snap
        self.error_code = 0


class StripOracle:
    def __init__(self, problem, strip, restatement, field_rows: np.ndarray):
        self.P = problem
        self.strip = strip
        self.orc = restatement
        self.nx = problem.nx
        self.ny = strip.ny_local
        self.field = np.array(field_rows, dtype=np.float64, copy=True)
        n = 4 * self.nx
        mk = lambda flag: torch.zeros(n, dtype=torch.float64) if flag else None  # noqa: E731
        self.send_s, self.recv_s = mk(strip.south_neighbor), mk(strip.south_neighbor)
        self.send_n, self.recv_n = mk(strip.north_neighbor), mk(strip.north_neighbor)
        self.slot = torch.zeros(2, dtype=torch.float64)
        self.local = abi.make_problem(2, self.nx, self.ny, problem.dx, problem.dy,
                                      a_g=problem.a_g, m_g=problem.m_g, cfl=problem.cfl,
                                      safety=problem.safety, gravity=problem.gravity,
                                      h_dry=problem.h_dry, bcs=list(problem.bc))
        self.launches = 0

    # interface --------------------------------------------------------------
    def exchange_tensors(self):
        return self.send_s, self.send_n, self.recv_s, self.recv_n

    def reduce_slot_tensor(self):
        return self.slot

    def _reduce(self):
        f = self.field.reshape(-1, 4)
        wet = f[:, 0] > self.P.h_dry
        self.wet = bool(wet.any())
        sx = sy = 0.0
        for c in f[wet]:
            h, u, v = c[0], c[1] / c[0], c[2] / c[0]
            sx = max(sx, self._axis_speed(h, u, v))
            sy = max(sy, self._axis_speed(h, v, u))
        self.slot[0] = sx
        self.slot[1] = sy
        f2 = self.field
        if self.send_s is not None:
            self.send_s.copy_(torch.from_numpy(np.ascontiguousarray(f2[0].T).reshape(-1)))
        if self.send_n is not None:
            self.send_n.copy_(torch.from_numpy(np.ascontiguousarray(f2[-1].T).reshape(-1)))

    def _axis_speed(self, h, un, ut):
        """axis_speed (src/stepper.cpp:30-36) with normal_flux_derivative
        (src/bedload.cpp:215-223); np.hypot is glibc's hypot."""
        P = self.P

        def abs_pow(au, q):
            return {0.0: 1.0, 1.0: au, 2.0: au * au, 3.0: au * au * au}.get(q, au ** q)

        def grass(u):
            return P.a_g * u * abs_pow(abs(u), P.m_g - 1.0)

        speed = float(np.hypot(un, ut))
        if speed <= 1e-10:
            dq = 0.0
        else:
            rate = grass(speed)
            drate = P.a_g * P.m_g * abs_pow(abs((h * speed) / h), P.m_g - 1.0) if h > 0 else 0.0
            ratio = un / speed
            dq = rate / speed + ratio * ratio * (drate - rate / speed)
        fluid = abs(un) + math.sqrt(P.gravity * h)
        solid = abs(un) + math.sqrt(un * un + P.gravity * dq)
        return solid if fluid < solid else fluid

    def begin(self, t_end=math.inf, max_steps=-1, snapshots=(), dt_cap=0):
        self.t_end, self.max_steps = t_end, max_steps
        self.snaps = sorted({s for s in snapshots if 0 < s <= t_end})
        self.t, self.steps, self.snap, self.state = 0.0, 0, 0, abi.STATE_RUNNING
        self._reduce()

    def step(self, n=1):
        for _ in range(n):
            self.launches += 1
            if self.state != abi.STATE_RUNNING:
                continue
            if not (self.t < self.t_end and (self.max_steps < 0 or self.steps < self.max_steps)):
                self.state = abi.STATE_DONE
                continue
            sx, sy = float(self.slot[0]), float(self.slot[1])
            raw = self.P.cfl * min(self.P.dx / sx, self.P.dy / sy)
            stop = min(self.snaps[self.snap], self.t_end) if self.snap < len(self.snaps) else self.t_end
            if stop - self.t <= raw:
                dt, t_new = stop - self.t, stop
            else:
                dt, t_new = raw, self.t + raw
            pad = np.zeros((self.ny + 2, self.nx + 2, 4))
            pad[1:-1, 1:-1] = self.field
            pad = self.orc.apply_bcs(self.local, pad)
            if self.recv_s is not None:
                pad[0, 1:-1] = self.recv_s.numpy().reshape(4, self.nx).T
            if self.recv_n is not None:
                pad[-1, 1:-1] = self.recv_n.numpy().reshape(4, self.nx).T
            self.field = self.orc.step_padded(self.local, pad, dt)[1:-1, 1:-1].copy()
            self.t, self.steps = t_new, self.steps + 1
            if self.snap < len(self.snaps) and self.t == self.snaps[self.snap]:
                self.snap += 1
                self.state = abi.STATE_PAUSED
            self._reduce()

    def status(self):
        return StripStatus(self.t, self.steps, self.state, self.snap)

    def resume(self):
        if self.state == abi.STATE_PAUSED:
            self.state = abi.STATE_RUNNING

    def launch_count(self):
        return self.launches

    def download(self, out=None):
        return self.field.copy()

    def close(self):
        pass
