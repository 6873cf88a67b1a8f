"""Snapshot CSV (write_snapshot / snapshot_to_string, reference
src/snapshot.cpp:50-93) formatted on the GPU, byte for byte.

CPU: the device formatter's "%.17g" (paper_1307_0491_b200/csrc/silt_csv.cuh,
built for the host by tests/cpp/fmt_harness.cpp) against glibc snprintf on
millions of doubles; the oracle's CSV restatement against the reference's
snapshot_to_string and a committed reference-made fixture; argument checks.
GPU: the device writer (host input, device input, solver planes, strip group,
file and memory sinks, chunked) against the restatement.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, ROOT, problem_from_meta
from paper_1307_0491_b200 import abi, scenarios

HARNESS = os.path.join(ROOT, "tests", "cpp", "_build", "libfmt_harness.so")


@pytest.fixture(scope="module")
def harness():
    if not os.path.exists(HARNESS):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "harness"], check=True)
    L = C.CDLL(HARNESS)
    L.fmt_g17_check.restype = C.c_longlong
    L.fmt_g17_check.argtypes = [C.c_void_p, C.c_longlong, C.POINTER(C.c_longlong)]
    L.fmt_g17_batch.argtypes = [C.c_void_p, C.c_longlong, C.c_char_p, C.c_longlong]
    return L


def _check(L, v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    first = C.c_longlong()
    bad = L.fmt_g17_check(v.ctypes.data, v.size, C.byref(first))
    if bad:
        buf = C.create_string_buffer(64)
        L.fmt_g17_batch(v[first.value:].ctypes.data, 1, buf, 64)
        pytest.fail(f"{bad} mismatches; first {v[first.value]!r}: {buf.value!r} "
                    f"vs {'%.17g' % v[first.value]!r}")


def edge_values() -> np.ndarray:
    """Specials, subnormals, powers of ten and two with their neighbours,
    17-digit rounding carries, exact ties."""
    out = [0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 5e-324, -5e-324,
           2.2250738585072014e-308, 2.225073858507201e-308, 1.7976931348623157e308,
           0.5, 0.1, 1 / 3, 1e16, 1e17, 99999999999999999.0, 1e-4, 1e-5, 9.99999999999999955e-5,
           2.0 ** 53, 2.0 ** 64, 123456789012345678.0]
    for e in range(-325, 309):
        x = 10.0 ** e if e >= -323 else 5e-324
        for d in (-2, -1, 0, 1, 2):
            y = x
            for _ in range(abs(d)):
                y = np.nextafter(y, np.inf if d > 0 else -np.inf)
            out += [y, -y]
    out += list(2.0 ** np.arange(-1074, 1024))
    out += list(np.arange(1, 50000, dtype=np.float64) * 1e12 + 0.5)
    return np.array(out)


def test_formatter_matches_glibc(harness):
    rng = np.random.default_rng(1307)
    bits = rng.integers(0, 2 ** 64, size=3_000_000, dtype=np.uint64)
    _check(harness, bits.view(np.float64))
    _check(harness, rng.uniform(-20, 20, 1_000_000))
    _check(harness, rng.standard_normal(500_000) * 1e-13)
    _check(harness, edge_values())


def _fields():
    """(problem, field, time) cases: 2D random bed, 1D dune, dry / stale cells."""
    out = []
    p, init, _ = scenarios.random_bed_2d(48, 32)
    out.append((p, init, 1.2345))
    p, init, _ = scenarios.dune_1d(cells=200)
    out.append((p, init, 0.0))
    p, init, _ = scenarios.random_bed_2d(20, 9)
    f = init.copy()
    f[0, :5, 0] = 0.0            # dry
    f[1, :5, 0] = 0.5e-8         # below h_dry with stale discharge
    f[2, :3, 1:3] = -0.0
    f[3, :4, 3] = -1e-300
    out.append((p, f, 7.0 / 3.0))
    return out


def test_restatement_csv_matches_reference(oracle_mod):
    if not oracle_mod.have_reference():
        pytest.skip("reference core not built")
    R, F = oracle_mod.restatement(), oracle_mod.reference()
    for p, f, t in _fields():
        assert R.snapshot_to_string(p, f, t) == F.snapshot_to_string(p, f, t)


def test_restatement_csv_matches_golden(restatement, golden):
    """tests/golden/snapshot_rand48x32.csv was written by the reference's
    snapshot_to_string (tests/golden/make_golden_csv.py)."""
    data, meta = golden
    m = meta["cases"]["rand48x32"]
    p = problem_from_meta(m)
    want = open(os.path.join(GOLDEN_DIR, "snapshot_rand48x32.csv"), "rb").read()
    assert restatement.snapshot_to_string(p, data["rand48x32_final"], m["t_final"]) == want


def test_abi_checks_rows_without_device():
    from paper_1307_0491_b200 import build, native
    build.build()
    p = abi.make_problem(2, 4, 3, 1.0, 1.0, a_g=0.1)
    with pytest.raises(native.InvalidArgument, match="rows outside"):
        native.snapshot_to_string(p, np.zeros((3, 4, 4)), 0.0, j0=2, rows=2)


# ------------------------------------------------------------------- GPU -----
@pytest.fixture(scope="module")
def N():
    from paper_1307_0491_b200 import native
    native.lib()
    return native


@pytest.mark.gpu
def test_gpu_csv_matches_restatement(N, restatement, tmp_path):
    for p, f, t in _fields():
        want = restatement.snapshot_to_string(p, f, t)
        assert N.snapshot_to_string(p, f, t) == want
        path = str(tmp_path / "s.csv")
        assert N.write_snapshot(p, f, t, path) == len(want)
        assert open(path, "rb").read() == want


@pytest.mark.gpu
def test_gpu_csv_edge_values(N, restatement):
    """Every edge value (bigint paths, subnormals, carries, specials) through the
    device formatter, laid out as a field."""
    v = edge_values()
    v = v[np.isfinite(v)]
    n = (v.size + 3) // 4 * 4
    v = np.resize(v, n).reshape(-1, 4)
    nx = 64
    rows = v.shape[0] // nx
    f = v[:rows * nx].reshape(rows, nx, 4).copy()
    f[..., 0] = np.abs(f[..., 0])
    p = abi.make_problem(2, nx, rows, 0.37, 1e-3, a_g=0.1)
    assert N.snapshot_to_string(p, f, 1e-300) == restatement.snapshot_to_string(p, f, 1e-300)


@pytest.mark.gpu
def test_gpu_csv_chunks_solver_and_group(N, restatement, golden, tmp_path, monkeypatch):
    """Chunked formatting (small chunks), straight from the solver's planes, and
    a 3-strip group writing one file, all equal to the restatement's bytes."""
    import torch
    from paper_1307_0491_b200.distributed import LocalStripGroup
    monkeypatch.setenv("SILT_CSV_CHUNK", "1000")
    data, meta = golden
    m = meta["cases"]["rand48x32"]
    p = problem_from_meta(m)
    f = data["rand48x32_final"]
    want = restatement.snapshot_to_string(p, f, m["t_final"])
    assert N.snapshot_to_string(p, f, m["t_final"]) == want
    d = torch.from_numpy(f.copy()).cuda()
    assert N.snapshot_to_string(p, d.data_ptr(), m["t_final"], rows=p.ny) == want
    s = N.Solver(p, variant=abi.VARIANT_STRICT)
    s.upload(data["rand48x32_init"])
    s.begin(max_steps=m["max_steps"])
    st = s.run(batch=16)
    path = str(tmp_path / "solver.csv")
    s.write_snapshot(st.t, path)
    s.close()
    assert open(path, "rb").read() == want
    g = LocalStripGroup(p, 3, devices=(0,), variant=abi.VARIANT_STRICT)
    g.upload(data["rand48x32_init"])
    g.begin(max_steps=m["max_steps"])
    st = g.run(batch=16)
    path = str(tmp_path / "group.csv")
    g.write_snapshot(st.t, path)
    g.close()
    assert open(path, "rb").read() == want


@pytest.mark.gpu
def test_gpu_async_csv_snapshots(N, restatement, golden, tmp_path):
    """silt_solver_capture_write: every snapshot of a run written as CSV in the
    background while the run continues; each file equals the restatement's CSV
    of the reference path run to that time (STRICT), and the run's end state
    is unaffected."""
    data, meta = golden
    m = meta["cases"]["rand48x32"]
    p = problem_from_meta(m)
    init = data["rand48x32_init"]
    T = m["t_final"]
    snaps = [0.2 * T, 0.2 * T + 1e-9, 0.6 * T]
    s = N.Solver(p, variant=abi.VARIANT_STRICT)
    s.upload(init)
    s.begin(max_steps=m["max_steps"] + len(snaps), snapshots=snaps)
    st = s.run_csv(str(tmp_path / "snap_%02d.csv"), batch=5)
    final = s.download()
    s.close()
    for k, t in enumerate(snaps):
        ref, rt, _, _ = restatement.run(p, init, t_end=t, snapshots=[x for x in snaps if x < t])
        assert rt == t
        want = restatement.snapshot_to_string(p, ref, t)
        assert open(tmp_path / f"snap_{k:02d}.csv", "rb").read() == want, k
    ref, rt, n, _ = restatement.run(p, init, max_steps=m["max_steps"] + len(snaps),
                                    snapshots=snaps)
    assert st.steps == n and np.array_equal(final, ref)


@pytest.mark.gpu
def test_gpu_capture_query_waits_for_the_writer(N, restatement, golden, tmp_path):
    """silt_solver_capture_query reports a background CSV snapshot as landed
    only once the file is completely written (then its bytes are final), and
    reports the writer's error (an unwritable path) instead of 'landed'."""
    import time
    data, meta = golden
    m = meta["cases"]["rand48x32"]
    p = problem_from_meta(m)
    init = data["rand48x32_init"]
    T = m["t_final"]
    s = N.Solver(p, variant=abi.VARIANT_STRICT)
    s.upload(init)
    s.begin(max_steps=m["max_steps"] + 2, snapshots=[0.3 * T, 0.7 * T])
    paths = [tmp_path / "a.csv", tmp_path / "missing_dir" / "b.csv"]
    results = []
    while True:
        s.step(4)
        st = s.status()
        if st.state == abi.STATE_PAUSED:
            k = len(results)
            field = s.download()
            s.capture_write(st.t, str(paths[k]))
            try:
                while not s.capture_query():
                    time.sleep(0.0005)
                results.append(("landed", st.t, field, paths[k].read_bytes()))
            except N.SiltRuntimeError as e:
                results.append(("error", st.t, field, str(e)))
            continue
        if st.state == abi.STATE_DONE:
            break
    s.capture_wait()
    s.close()
    kind, t, field, got = results[0]
    assert kind == "landed" and got == restatement.snapshot_to_string(p, field, t)
    assert results[1][0] == "error"
