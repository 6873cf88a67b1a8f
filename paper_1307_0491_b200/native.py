"""ctypes binding of libsilt_b200.so (include/silt_cuda.h).

The CUDA library is the only compute path: there is no CPU fallback.  If the
library is missing, importing the bindings raises ``SiltLibraryMissing``.
Status codes map onto the reference's exception classes:
SILT_ERR_INVALID -> InvalidArgument (std::invalid_argument),
SILT_ERR_RUNTIME -> SiltRuntimeError (std::runtime_error).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi
from .abi import SiltExchange, SiltProblem, SiltRunPlan, SiltStatus, SiltStrip

LIB_PATH = os.environ.get(
    "SILT_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libsilt_b200.so"))


class SiltLibraryMissing(ImportError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class SiltRuntimeError(RuntimeError):
    """std::runtime_error in the reference."""


class SiltCudaError(RuntimeError):
    pass


_lib = None

_P = C.POINTER(SiltProblem)
_D = C.POINTER(C.c_double)
_VP = C.c_void_p


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SiltLibraryMissing(
            f"{LIB_PATH} not built; run `python -m paper_1307_0491_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    sigs = {
        "silt_abi_version": ([], C.c_int),
        "silt_abi_sizes": ([C.POINTER(C.c_int64), C.c_int], C.c_int),
        "silt_last_error": ([], C.c_char_p),
        "silt_device_count": ([C.POINTER(C.c_int)], C.c_int),
        "silt_solver_create": ([_P, C.POINTER(SiltStrip), C.c_int, C.c_int, C.POINTER(_VP)], C.c_int),
        "silt_solver_destroy": ([_VP], C.c_int),
        "silt_solver_set_stream": ([_VP, _VP], C.c_int),
        "silt_solver_upload": ([_VP, _D], C.c_int),
        "silt_solver_download": ([_VP, _D], C.c_int),
        "silt_solver_upload_device": ([_VP, _VP], C.c_int),
        "silt_solver_download_device": ([_VP, _VP], C.c_int),
        "silt_solver_set_ghosts": ([_VP, _D, _D, _D, _D], C.c_int),
        "silt_solver_begin": ([_VP, C.POINTER(SiltRunPlan)], C.c_int),
        "silt_solver_step": ([_VP, C.c_int], C.c_int),
        "silt_solver_step_fixed": ([_VP, C.c_double], C.c_int),
        "silt_solver_status": ([_VP, C.POINTER(SiltStatus)], C.c_int),
        "silt_solver_resume": ([_VP], C.c_int),
        "silt_solver_dt_log": ([_VP, _D, C.c_int64], C.c_int),
        "silt_solver_cfl_dt": ([_VP, _D], C.c_int),
        "silt_solver_reduce_slot": ([_VP, C.POINTER(_VP)], C.c_int),
        "silt_solver_exchange_ptrs": ([_VP, C.POINTER(SiltExchange)], C.c_int),
        "silt_solver_launch_count": ([_VP, C.POINTER(C.c_int64)], C.c_int),
        "silt_run": ([_P, _D, C.POINTER(SiltRunPlan), C.c_int, _D, _D, C.c_int64,
                      C.POINTER(SiltStatus)], C.c_int),
        "silt_cfl_dt": ([_P, _D, C.c_int, _D], C.c_int),
        "silt_step_padded": ([_P, _D, C.c_double, C.c_int], C.c_int),
        "silt_riemann_batch": ([_P, _D, _D, C.c_int64, C.c_int, C.c_int, _D], C.c_int),
        "silt_law_batch": ([_P, _D, C.c_int64, C.c_int, _D], C.c_int),
        "silt_selftest_math": ([_D, _D, C.c_int64, _D], C.c_int),
        "silt_group_create": ([_P, C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int,
                               C.POINTER(_VP)], C.c_int),
        "silt_group_destroy": ([_VP], C.c_int),
        "silt_group_upload": ([_VP, _D], C.c_int),
        "silt_group_download": ([_VP, _D], C.c_int),
        "silt_group_begin": ([_VP, C.POINTER(SiltRunPlan)], C.c_int),
        "silt_group_step": ([_VP, C.c_int], C.c_int),
        "silt_group_status": ([_VP, C.POINTER(SiltStatus)], C.c_int),
        "silt_group_resume": ([_VP], C.c_int),
        "silt_group_dt_log": ([_VP, _D, C.c_int64], C.c_int),
        "silt_group_timing": ([_VP, C.c_int, _D], C.c_int),
        "silt_solver_timing": ([_VP, C.c_int, _D], C.c_int),
        "silt_group_capture_resume": ([_VP, _D], C.c_int),
        "silt_group_capture_wait": ([_VP], C.c_int),
        "silt_solver_capture_resume": ([_VP, _D], C.c_int),
        "silt_solver_capture_wait": ([_VP], C.c_int),
        "silt_solver_capture_query": ([_VP, C.POINTER(C.c_int)], C.c_int),
        "silt_solver_capture_write": ([_VP, C.c_double, C.c_char_p, C.c_int], C.c_int),
        "silt_host_alloc": ([C.c_int64, C.POINTER(_VP)], C.c_int),
        "silt_host_free": ([_VP], C.c_int),
        "silt_solver_step_split_ok": ([_VP, C.POINTER(C.c_int)], C.c_int),
        "silt_solver_p2p_export": ([_VP, C.c_void_p], C.c_int),
        "silt_solver_p2p_connect": ([_VP, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int], C.c_int),
        "silt_solver_p2p_step": ([_VP, C.c_int], C.c_int),
        "silt_solver_step_part": ([_VP, C.c_int], C.c_int),
        "silt_snapshot_to_string": ([_P, _VP, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                     C.c_char_p, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
        "silt_write_snapshot": ([_P, _VP, C.c_int64, C.c_int64, C.c_double, C.c_char_p,
                                 C.c_int, C.POINTER(C.c_int64)], C.c_int),
        "silt_solver_write_snapshot": ([_VP, C.c_double, C.c_char_p, C.c_int,
                                        C.POINTER(C.c_int64)], C.c_int),
        "silt_group_write_snapshot": ([_VP, C.c_double, C.c_char_p, C.POINTER(C.c_int64)],
                                      C.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.silt_abi_version() != abi.SILT_ABI_VERSION:
        raise SiltLibraryMissing("libsilt_b200.so ABI version mismatch; rebuild")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == abi.SILT_OK:
        return
    msg = lib().silt_last_error().decode()
    if rc == abi.SILT_ERR_INVALID:
        raise InvalidArgument(msg)
    if rc == abi.SILT_ERR_RUNTIME:
        raise SiltRuntimeError(msg)
    if rc == abi.SILT_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise SiltCudaError(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _plan(t_end: float, max_steps: int, snapshots, dt_cap: int):
    snaps = np.ascontiguousarray(np.asarray(snapshots, dtype=np.float64).reshape(-1))
    plan = SiltRunPlan(float(t_end), int(max_steps),
                       _dp(snaps) if snaps.size else None, int(snaps.size), int(dt_cap))
    return plan, snaps


class PinnedField:
    """Page-locked host field (silt_host_alloc) viewed as a (ny, nx, 4) array."""

    def __init__(self, ny: int, nx: int):
        self.L = lib()
        self.ptr = _VP()
        n = ny * nx * 4
        check(self.L.silt_host_alloc(n * 8, C.byref(self.ptr)))
        self.array = np.ctypeslib.as_array((C.c_double * n).from_address(self.ptr.value))
        self.array = self.array.reshape(ny, nx, 4)

    def close(self):
        if self.ptr:
            self.array = None
            self.L.silt_host_free(self.ptr)
            self.ptr = _VP()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _run_loop(step, status, resume, download, capture, wait, batch, on_snapshot,
              async_snapshots, shape):
    """The run loop shared by Solver and LocalStripGroup (src/parallel.cpp:208-259).

    Synchronous snapshots: download, call on_snapshot(t, field), resume.
    Asynchronous snapshots (``async_snapshots=True``): capture into a pinned
    buffer and resume at once; on_snapshot(t, view) runs when the copy has
    landed (at the latest before the next capture and at the end), while the
    device keeps stepping.  The view is valid during the callback only, like
    the reference's ``const Field&``.
    """
    pinned = None
    pending = None
    try:
        while True:
            step(batch)
            st = status()
            if st.state == abi.STATE_PAUSED:
                if on_snapshot is None:
                    resume()
                elif not async_snapshots:
                    on_snapshot(st.t, download())
                    resume()
                else:
                    if pending is not None:
                        wait()
                        on_snapshot(pending, pinned.array)
                    if pinned is None:
                        pinned = PinnedField(*shape)
                    capture(pinned.array)
                    pending = st.t
                continue
            if st.state == abi.STATE_DONE:
                if pending is not None:
                    wait()
                    on_snapshot(pending, pinned.array)
                return st
    finally:
        if pinned is not None:
            try:
                wait()  # no copy may still target the buffer when it is freed
            finally:
                pinned.close()


class Solver:
    """One strip (or the whole grid) resident on one GPU."""

    def __init__(self, problem: SiltProblem, strip: SiltStrip | None = None, device: int = 0,
                 variant: int = abi.VARIANT_FAST):
        self.L = lib()
        self.problem = problem
        self.h = _VP()
        check(self.L.silt_solver_create(C.byref(problem), C.byref(strip) if strip else None,
                                        device, variant, C.byref(self.h)))
        ny = 1 if problem.dim == 1 else problem.ny
        self.nx = problem.nx
        self.ny = strip.ny_local if strip else ny

    def close(self):
        if self.h:
            self.L.silt_solver_destroy(self.h)
            self.h = _VP()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # data movement ---------------------------------------------------------
    def upload(self, field: np.ndarray):
        field = np.ascontiguousarray(field, dtype=np.float64)
        assert field.size == 4 * self.nx * self.ny
        check(self.L.silt_solver_upload(self.h, _dp(field)))

    def upload_device(self, ptr: int):
        """Device AoS copy on the solver's stream.  The caller orders the
        producer of ``ptr`` first (e.g. torch.cuda.current_stream().synchronize())."""
        check(self.L.silt_solver_upload_device(self.h, ptr))

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.ny, self.nx, 4))
        check(self.L.silt_solver_download(self.h, _dp(out)))
        return out

    def download_device(self, ptr: int):
        check(self.L.silt_solver_download_device(self.h, ptr))

    def set_stream(self, stream_ptr: int):
        check(self.L.silt_solver_set_stream(self.h, stream_ptr))

    # run control -------------------------------------------------------------
    def begin(self, t_end: float = np.inf, max_steps: int = -1, snapshots=(), dt_cap: int = 0):
        plan, keep = _plan(t_end, max_steps, snapshots, dt_cap)
        check(self.L.silt_solver_begin(self.h, C.byref(plan)))
        del keep

    def step(self, n: int = 1):
        check(self.L.silt_solver_step(self.h, int(n)))

    # multi-process peer-memory exchange (silt_solver_p2p_*)
    def p2p_export(self) -> bytes:
        buf = C.create_string_buffer(200)
        check(self.L.silt_solver_p2p_export(self.h, buf))
        return buf.raw[:200]

    def p2p_connect(self, rank: int, world: int, handles, south, north):
        blob = b"".join(handles)
        check(self.L.silt_solver_p2p_connect(self.h, rank, world, blob,
                                             -1 if south is None else south,
                                             -1 if north is None else north))

    def p2p_step(self, n: int = 1):
        check(self.L.silt_solver_p2p_step(self.h, int(n)))

    def split_ok(self) -> bool:
        ok = C.c_int(0)
        check(self.L.silt_solver_step_split_ok(self.h, C.byref(ok)))
        return bool(ok.value)

    def step_part(self, part: int):
        """Part 1 (boundary row blocks) or 2 (interior, ends the step) of a split step."""
        check(self.L.silt_solver_step_part(self.h, int(part)))

    def step_fixed(self, dt: float):
        check(self.L.silt_solver_step_fixed(self.h, float(dt)))

    def status(self) -> SiltStatus:
        st = SiltStatus()
        check(self.L.silt_solver_status(self.h, C.byref(st)))
        return st

    def resume(self):
        check(self.L.silt_solver_resume(self.h))

    def dt_log(self, n: int) -> np.ndarray:
        out = np.empty(n)
        check(self.L.silt_solver_dt_log(self.h, _dp(out), int(n)))
        return out

    def cfl_dt(self) -> float:
        dt = C.c_double()
        check(self.L.silt_solver_cfl_dt(self.h, C.byref(dt)))
        return dt.value

    def reduce_slot(self) -> int:
        p = _VP()
        check(self.L.silt_solver_reduce_slot(self.h, C.byref(p)))
        return p.value

    def exchange_ptrs(self) -> SiltExchange:
        ex = SiltExchange()
        check(self.L.silt_solver_exchange_ptrs(self.h, C.byref(ex)))
        return ex

    def launch_count(self) -> int:
        n = C.c_int64()
        check(self.L.silt_solver_launch_count(self.h, C.byref(n)))
        return n.value

    def capture_resume(self, out: np.ndarray):
        """Asynchronous snapshot of a paused run into ``out`` (pinned memory
        overlaps the copy with the next steps); see silt_solver_capture_resume."""
        assert out.flags.c_contiguous and out.size == 4 * self.nx * self.ny
        check(self.L.silt_solver_capture_resume(self.h, _dp(out)))

    def capture_wait(self):
        check(self.L.silt_solver_capture_wait(self.h))

    def capture_query(self) -> bool:
        """True once the last capture (device copy, or a background CSV write)
        has fully landed; raises the background writer's error."""
        landed = C.c_int(0)
        check(self.L.silt_solver_capture_query(self.h, C.byref(landed)))
        return bool(landed.value)

    def capture_write(self, time: float, path: str, append: bool = False):
        """CSV snapshot of a paused run, written in the background while the run
        continues (silt_solver_capture_write); capture_wait() joins it."""
        check(self.L.silt_solver_capture_write(self.h, float(time), os.fsencode(path),
                                               int(append)))

    def run_csv(self, pattern: str, batch: int = 32) -> SiltStatus:
        """Advance until DONE, writing every snapshot as CSV (pattern % index,
        e.g. 'out/snap_%04d.csv') in the background."""
        k = 0
        try:
            while True:
                self.step(batch)
                st = self.status()
                if st.state == abi.STATE_PAUSED:
                    self.capture_write(st.t, pattern % k)
                    k += 1
                    continue
                if st.state == abi.STATE_DONE:
                    return st
        finally:
            self.capture_wait()

    def write_snapshot(self, time: float, path: str, append: bool = False) -> int:
        """CSV of the current state (write_snapshot) formatted on the device."""
        n = C.c_int64(0)
        check(self.L.silt_solver_write_snapshot(self.h, float(time), os.fsencode(path),
                                                int(append), C.byref(n)))
        return n.value

    def run(self, batch: int = 32, on_snapshot=None, async_snapshots: bool = False) -> SiltStatus:
        """Advance until DONE; PAUSED snapshots call on_snapshot(t, field)."""
        return _run_loop(self.step, self.status, self.resume, self.download,
                         self.capture_resume, self.capture_wait, batch, on_snapshot,
                         async_snapshots, (self.ny, self.nx))


# ---- one-shot conveniences (mirror the reference free functions) -------------
def run(problem: SiltProblem, init: np.ndarray, *, t_end: float = np.inf, max_steps: int = -1,
        snapshots=(), variant: int = abi.VARIANT_FAST, dt_log: bool = True):
    """run_serial on one GPU: returns (final field, t, steps, dt log)."""
    L = lib()
    init = np.ascontiguousarray(init, dtype=np.float64)
    out = np.empty_like(init)
    cap = (max_steps if max_steps >= 0 else 1 << 20) if dt_log else 0
    log = np.empty(max(cap, 1))
    plan, keep = _plan(t_end, max_steps, snapshots, cap)
    st = SiltStatus()
    check(L.silt_run(C.byref(problem), _dp(init), C.byref(plan), variant, _dp(out),
                     _dp(log) if dt_log else None, cap, C.byref(st)))
    del keep
    return out, st.t, st.steps, (log[:min(st.steps, cap)].copy() if dt_log else None)


def cfl_dt(problem: SiltProblem, field: np.ndarray, variant: int = abi.VARIANT_FAST) -> float:
    field = np.ascontiguousarray(field, dtype=np.float64)
    dt = C.c_double()
    check(lib().silt_cfl_dt(C.byref(problem), _dp(field), variant, C.byref(dt)))
    return dt.value


def step_padded(problem: SiltProblem, padded: np.ndarray, dt: float,
                variant: int = abi.VARIANT_FAST) -> np.ndarray:
    padded = np.array(padded, dtype=np.float64, order="C", copy=True)
    check(lib().silt_step_padded(C.byref(problem), _dp(padded), float(dt), variant))
    return padded


def faces(problem: SiltProblem, left: np.ndarray, right: np.ndarray, axis: int,
          variant: int = abi.VARIANT_FAST) -> np.ndarray:
    left = np.ascontiguousarray(left, dtype=np.float64).reshape(-1, 4)
    right = np.ascontiguousarray(right, dtype=np.float64).reshape(-1, 4)
    out = np.empty((left.shape[0], 5))
    check(lib().silt_riemann_batch(C.byref(problem), _dp(left), _dp(right), left.shape[0],
                                   axis, variant, _dp(out)))
    return out


def _field_ptr(field, problem: SiltProblem, rows):
    """(pointer, rows) of a host ndarray or a device pointer (int, needs rows)."""
    if isinstance(field, np.ndarray):
        field = np.ascontiguousarray(field, dtype=np.float64)
        n = field.size // (4 * problem.nx)
        return field, field.ctypes.data, (n if rows is None else rows)
    if rows is None:
        raise ValueError("rows is required for a device pointer")
    return None, int(field), rows


def snapshot_to_string(problem: SiltProblem, field, time: float, *, j0: int = 0,
                       rows: int | None = None, header: bool = True) -> bytes:
    """snapshot_to_string (reference src/snapshot.cpp:50-84), formatted on the GPU.
    ``field``: AoS rows [j0, j0 + rows) — a numpy array or a device pointer."""
    keep, ptr, rows = _field_ptr(field, problem, rows)
    n = C.c_int64(0)
    rc = lib().silt_snapshot_to_string(C.byref(problem), ptr, j0, rows, float(time),
                                       int(header), None, 0, C.byref(n))
    if rc not in (abi.SILT_OK, abi.SILT_ERR_INVALID) or (rc and n.value == 0):
        check(rc)
    buf = C.create_string_buffer(max(n.value, 1))
    check(lib().silt_snapshot_to_string(C.byref(problem), ptr, j0, rows, float(time),
                                        int(header), buf, n.value, C.byref(n)))
    del keep
    return buf.raw[:n.value]


def write_snapshot(problem: SiltProblem, field, time: float, path: str, *, j0: int = 0,
                   rows: int | None = None, append: bool = False) -> int:
    """write_snapshot (reference src/snapshot.cpp:86-93), formatted on the GPU;
    returns the bytes written."""
    keep, ptr, rows = _field_ptr(field, problem, rows)
    n = C.c_int64(0)
    check(lib().silt_write_snapshot(C.byref(problem), ptr, j0, rows, float(time),
                                    os.fsencode(path), int(append), C.byref(n)))
    del keep
    return n.value


def law_terms(problem: SiltProblem, states: np.ndarray,
              variant: int = abi.VARIANT_FAST) -> np.ndarray:
    """(n, 2): normal_flux, normal_flux_derivative of states (n, 3) = (h, u_n, u_t)."""
    states = np.ascontiguousarray(states, dtype=np.float64).reshape(-1, 3)
    out = np.empty((states.shape[0], 2))
    check(lib().silt_law_batch(C.byref(problem), _dp(states), states.shape[0], variant,
                               _dp(out)))
    return out


def selftest_math(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """(n, 4): fast rcp, IEEE rcp, strict (glibc) hypot, sqrt — on the device."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty((x.size, 4))
    check(lib().silt_selftest_math(_dp(x), _dp(y), x.size, _dp(out)))
    return out
