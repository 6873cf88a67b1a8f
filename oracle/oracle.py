"""ctypes access to the parity CHECKERS — TEST INFRASTRUCTURE ONLY.

Two libraries with the same entry points:
  * ``restatement()``  -> oracle/_build/libsilt_oracle.so (our C restatement,
    oracle/silt_oracle.c)
  * ``reference()``    -> oracle/_ref/libsilt_ref.so (the unmodified reference
    core compiled from /root/reference by oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_1307_0491_b200.abi import SiltProblem  # noqa: E402

RESTATEMENT_SO = os.path.join(_HERE, "_build", "libsilt_oracle.so")
REFERENCE_SO = os.path.join(_HERE, "_ref", "libsilt_ref.so")

_P = C.POINTER(SiltProblem)
_D = C.POINTER(C.c_double)
_I64 = C.c_int64


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(reference: bool = True) -> None:
    """Build the checkers (make -C oracle)."""
    targets = ["oracle"] + (["ref"] if reference else [])
    subprocess.run(["make", "-s", "-C", _HERE] + targets, check=True)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


class CpuSolver:
    """Uniform wrapper over one checker library (prefix ``orc`` or ``ref``)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        L = self.lib
        f = getattr(L, f"{prefix}_last_error")
        f.restype = C.c_char_p
        self._err = f
        g = getattr(L, f"{prefix}_run")
        g.argtypes = [_P, _D, C.c_double, _I64, _D, C.c_int, _D, _D, _I64,
                      C.POINTER(_I64), _D]
        g.restype = C.c_int
        self._run = g
        g = getattr(L, f"{prefix}_cfl_dt")
        g.argtypes = [_P, _D, _D]
        self._cfl = g
        g = getattr(L, f"{prefix}_step_padded")
        g.argtypes = [_P, _D, C.c_double]
        self._step = g
        g = getattr(L, f"{prefix}_apply_bcs")
        g.argtypes = [_P, _D]
        self._bcs = g
        g = getattr(L, f"{prefix}_face_batch")
        g.argtypes = [_P, _D, _D, _I64, C.c_int, _D, _D]
        self._face = g
        g = getattr(L, f"{prefix}_riemann")
        g.argtypes = [_D, _D, C.c_double, C.c_double, C.c_double, _D]
        self._riemann = g
        g = getattr(L, f"{prefix}_relax")
        g.argtypes = [_P, _D, _D, C.c_int, _D]
        self._relax = g
        g = getattr(L, f"{prefix}_law_eval")
        g.argtypes = [_P, _D, _I64, _D]
        self._law = g
        g = getattr(L, f"{prefix}_snapshot_to_string")
        g.argtypes = [_P, _D, C.c_double, C.c_char_p, _I64, C.POINTER(_I64)]
        self._snap = g
        g = getattr(L, f"{prefix}_shields_flux")
        g.argtypes = [C.c_int, _D, _D, _I64, _D]
        self._shields = g
        if prefix == "ref":
            g = L.ref_run_parallel
            g.argtypes = [_P, _D, C.c_double, _I64, C.c_int, C.c_int, _D,
                          C.POINTER(_I64), _D, _D, _D]
            self._runp = g
            g = L.ref_build_scenario
            g.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, _P, _D, C.POINTER(_I64), _D]
            g.restype = C.c_int
            self._build = g
            g = L.ref_run_snaps
            g.argtypes = [_P, _D, C.c_double, _D, C.c_int, _D, C.POINTER(C.c_int), _D,
                          C.POINTER(_I64)]
            g.restype = C.c_int
            self._runs = g
            g = L.ref_run_blocks
            g.argtypes = [_P, _D, _I64, C.c_int, C.c_int, _D, _D, C.POINTER(_I64), _D]
            g.restype = C.c_int
            self._runb = g

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._err().decode())

    def run(self, problem: SiltProblem, init: np.ndarray, *, t_end: float = np.inf,
            max_steps: int = -1, snapshots=(), dt_log: bool = True):
        init = np.ascontiguousarray(init, dtype=np.float64)
        out = np.empty_like(init)
        cap = max(int(max_steps), 0) if max_steps >= 0 else 1 << 20
        log = np.zeros(cap if dt_log else 1)
        snaps = np.ascontiguousarray(np.asarray(snapshots, dtype=np.float64).reshape(-1))
        steps = _I64(0)
        t = C.c_double(0)
        self._check(self._run(C.byref(problem), _dp(init), float(t_end), int(max_steps),
                              _dp(snaps) if snaps.size else None, int(snaps.size),
                              _dp(out), _dp(log) if dt_log else None,
                              cap if dt_log else 0, C.byref(steps), C.byref(t)))
        n = steps.value
        return out, t.value, n, (log[:min(n, cap)].copy() if dt_log else None)

    def run_parallel(self, problem, init, px, py, *, t_end=np.inf, max_steps=-1,
                     want_field=True):
        init = np.ascontiguousarray(init, dtype=np.float64)
        out = np.empty_like(init) if want_field else None
        steps = _I64(0)
        t = C.c_double(0)
        comp = C.c_double(0)
        wall = C.c_double(0)
        self._check(self._runp(C.byref(problem), _dp(init), float(t_end), int(max_steps),
                               int(px), int(py), _dp(out) if want_field else None,
                               C.byref(steps), C.byref(t), C.byref(comp), C.byref(wall)))
        return out, t.value, steps.value, comp.value, wall.value

    def run_blocks(self, problem, init, max_steps: int, py: int, threads: int):
        """run_parallel's loop on Topology{1, py} through the public API with a
        dt log (ref_run_blocks): (field, t, steps, dt_log)."""
        init = np.ascontiguousarray(init, dtype=np.float64)
        out = np.empty_like(init)
        log = np.zeros(max(int(max_steps), 1))
        steps = _I64(0)
        t = C.c_double(0)
        self._check(self._runb(C.byref(problem), _dp(init), int(max_steps), int(py),
                               int(threads), _dp(out), _dp(log), C.byref(steps),
                               C.byref(t)))
        return out, t.value, steps.value, log[:steps.value].copy()

    def build_scenario(self, name: str, cells_x: int = 0, cells_y: int = 0, a_g: float = 1.0):
        """The reference's bundled scenario (build_scenario / build_bump_2d):
        (problem, AoS initial field (ny, nx, 4), t_end)."""
        p = SiltProblem()
        n = _I64(0)
        t_end = C.c_double(0)
        self._check(self._build(name.encode(), cells_x, cells_y, a_g, C.byref(p), None,
                                C.byref(n), C.byref(t_end)))
        init = np.empty((p.ny, p.nx, 4))
        self._check(self._build(name.encode(), cells_x, cells_y, a_g, C.byref(p), _dp(init),
                                C.byref(n), C.byref(t_end)))
        return p, init, t_end.value

    def run_snaps(self, problem, init, t_end: float, times):
        """run_serial with snapshot times: (list of landed fields, t, steps)."""
        init = np.ascontiguousarray(init, dtype=np.float64)
        times = np.ascontiguousarray(np.asarray(times, dtype=np.float64))
        out = np.empty((len(times),) + init.shape)
        landed = C.c_int(0)
        t = C.c_double(0)
        steps = _I64(0)
        self._check(self._runs(C.byref(problem), _dp(init), float(t_end), _dp(times), len(times),
                               _dp(out), C.byref(landed), C.byref(t), C.byref(steps)))
        return [out[k] for k in range(min(landed.value, len(times)))], t.value, steps.value

    def cfl_dt(self, problem, field) -> float:
        field = np.ascontiguousarray(field, dtype=np.float64)
        dt = C.c_double(0)
        self._check(self._cfl(C.byref(problem), _dp(field), C.byref(dt)))
        return dt.value

    def step_padded(self, problem, padded, dt) -> np.ndarray:
        padded = np.array(padded, dtype=np.float64, order="C", copy=True)
        self._check(self._step(C.byref(problem), _dp(padded), float(dt)))
        return padded

    def apply_bcs(self, problem, padded) -> np.ndarray:
        padded = np.array(padded, dtype=np.float64, order="C", copy=True)
        self._check(self._bcs(C.byref(problem), _dp(padded)))
        return padded

    def faces(self, problem, left, right, axis: int):
        left = np.ascontiguousarray(left, dtype=np.float64).reshape(-1, 4)
        right = np.ascontiguousarray(right, dtype=np.float64).reshape(-1, 4)
        n = left.shape[0]
        out = np.empty((n, 5))
        info = np.empty((n, 4))
        self._check(self._face(C.byref(problem), _dp(left), _dp(right), n, axis,
                               _dp(out), _dp(info)))
        return out, info

    def riemann(self, l5, r5, a, b, g=9.81) -> np.ndarray:
        l5 = np.ascontiguousarray(l5, dtype=np.float64)
        r5 = np.ascontiguousarray(r5, dtype=np.float64)
        out = np.empty(42)
        self._check(self._riemann(_dp(l5), _dp(r5), a, b, g, _dp(out)))
        return out

    def relax(self, problem, lc, rc, axis: int) -> np.ndarray:
        lc = np.ascontiguousarray(lc, dtype=np.float64)
        rc = np.ascontiguousarray(rc, dtype=np.float64)
        out = np.empty(12)
        self._check(self._relax(C.byref(problem), _dp(lc), _dp(rc), axis, _dp(out)))
        return out

    def law_eval(self, problem, states) -> np.ndarray:
        """(n, 6) law probes of states (n, 3) = (h, u_n, u_t): dimensional_flux,
        dqs_du, normal_flux, normal_flux_derivative, shields_stress, friction_slope."""
        states = np.ascontiguousarray(states, dtype=np.float64).reshape(-1, 3)
        out = np.empty((states.shape[0], 6))
        self._check(self._law(C.byref(problem), _dp(states), states.shape[0], _dp(out)))
        return out

    def snapshot_to_string(self, problem, field, time: float) -> bytes:
        """snapshot_to_string (src/snapshot.cpp:50-84) of a whole-grid field."""
        field = np.ascontiguousarray(field, dtype=np.float64)
        n = _I64(0)
        self._check(self._snap(C.byref(problem), _dp(field), float(time), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        self._check(self._snap(C.byref(problem), _dp(field), float(time), buf, n.value,
                               C.byref(n)))
        return buf.raw[:n.value]

    def shields_flux(self, formula: int, tau, tau_cr) -> np.ndarray:
        """(n, 2): shields_flux, shields_flux_derivative."""
        tau = np.ascontiguousarray(tau, dtype=np.float64).ravel()
        tau_cr = np.ascontiguousarray(np.broadcast_to(tau_cr, tau.shape), dtype=np.float64)
        out = np.empty((tau.size, 2))
        self._check(self._shields(formula, _dp(tau), _dp(tau_cr), tau.size, _dp(out)))
        return out


_cache: dict = {}


def restatement() -> CpuSolver:
    if "orc" not in _cache:
        _cache["orc"] = CpuSolver(RESTATEMENT_SO, "orc")
    return _cache["orc"]


def reference() -> CpuSolver:
    if "ref" not in _cache:
        _cache["ref"] = CpuSolver(REFERENCE_SO, "ref")
    return _cache["ref"]


def have_reference() -> bool:
    return os.path.exists(REFERENCE_SO)


def padded(field: np.ndarray) -> np.ndarray:
    """Interior (ny, nx, 4) -> PaddedField layout (ny+2, nx+2, 4), zero ghosts
    (include/silt/stepper.hpp:14-32)."""
    ny, nx, _ = field.shape
    p = np.zeros((ny + 2, nx + 2, 4))
    p[1:-1, 1:-1] = field
    return p
