"""ctypes mirror of include/silt_cuda.h (the C-ABI drop-in boundary).

Only structure layouts and constants live here; loading the CUDA library is
paper_1307_0491_b200.native's job.  The reference types these structures stand
for are cited in include/silt_cuda.h.
"""
from __future__ import annotations

import ctypes as C
import math

SILT_ABI_VERSION = 2

SILT_OK = 0
SILT_ERR_INVALID = 1
SILT_ERR_RUNTIME = 2
SILT_ERR_CUDA = 3
SILT_ERR_UNSUPPORTED = 4

BC_INFLOW = 0
BC_OUTFLOW = 1
BC_WALL = 2
BC_PERIODIC = 3
BC_GIVEN = 4

WEST, EAST, SOUTH, NORTH = 0, 1, 2, 3

VARIANT_FAST = 0
VARIANT_STRICT = 1

LAW_GRASS = 0
LAW_SHIELDS = 1

# ShieldsFormula / FrictionModel in the reference's enum order
# (include/silt/bedload.hpp:12-23); keys are the reference's CLI/config names
# (src/config.cpp:228-267).
SHIELDS_FORMULAS = {"mpm": 0, "flvb": 1, "nielsen": 2, "ribberink": 3, "camenen": 4}
FRICTION_MODELS = {"darcy-weisbach": 0, "manning": 1}

STATE_RUNNING = 0
STATE_DONE = 1
STATE_PAUSED = 2
STATE_FAILED = 3


class SiltBC(C.Structure):
    _fields_ = [("type", C.c_int32), ("supercritical", C.c_int32),
                ("q0", C.c_double), ("h0", C.c_double)]


class SiltProblem(C.Structure):
    _fields_ = [("dim", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
                ("law_kind", C.c_int32),
                ("dx", C.c_double), ("dy", C.c_double),
                ("gravity", C.c_double), ("h_dry", C.c_double),
                ("a_g", C.c_double), ("m_g", C.c_double),
                ("shields_formula", C.c_int32), ("friction_model", C.c_int32),
                ("tau_cr", C.c_double), ("grain_diameter", C.c_double),
                ("rel_density", C.c_double), ("friction_coef", C.c_double),
                ("cfl", C.c_double), ("safety", C.c_double),
                ("bc", SiltBC * 4)]


class SiltStrip(C.Structure):
    _fields_ = [("j0", C.c_int32), ("ny_local", C.c_int32),
                ("south_neighbor", C.c_int32), ("north_neighbor", C.c_int32)]


class SiltRunPlan(C.Structure):
    _fields_ = [("t_end", C.c_double), ("max_steps", C.c_int64),
                ("snapshot_times", C.POINTER(C.c_double)),
                ("n_snapshots", C.c_int32),
                ("dt_log_capacity", C.c_int64)]


class SiltStatus(C.Structure):
    _fields_ = [("t", C.c_double), ("steps", C.c_int64), ("state", C.c_int32),
                ("error_code", C.c_int32), ("last_dt", C.c_double),
                ("snapshot_index", C.c_int32), ("pad_", C.c_int32)]


class SiltExchange(C.Structure):
    _fields_ = [("send_south", C.c_void_p), ("send_north", C.c_void_p),
                ("recv_south", C.c_void_p), ("recv_north", C.c_void_p),
                ("row_doubles", C.c_int64)]


def bc(kind: str = "outflow", q0: float = 0.0, h0: float = 0.0,
       supercritical: bool = False) -> SiltBC:
    """BoundarySpec factories (reference include/silt/scenarios.hpp:24-35)."""
    t = {"inflow": BC_INFLOW, "outflow": BC_OUTFLOW, "wall": BC_WALL,
         "periodic": BC_PERIODIC, "given": BC_GIVEN}[kind]
    return SiltBC(t, 1 if supercritical else 0, float(q0), float(h0))


def make_problem(dim: int, nx: int, ny: int, dx: float, dy: float, *,
                 a_g: float, m_g: float = 3.0, cfl: float = 0.5,
                 safety: float = 1.05, gravity: float = 9.81,
                 h_dry: float = 1e-8, bcs=None) -> SiltProblem:
    p = SiltProblem()
    p.dim = dim
    p.nx = nx
    p.ny = 1 if dim == 1 else ny
    p.law_kind = 0
    p.dx = dx
    p.dy = 1.0 if dim == 1 else dy
    p.gravity = gravity
    p.h_dry = h_dry
    p.a_g = a_g
    p.m_g = m_g
    p.cfl = cfl
    p.safety = safety
    bcs = bcs or [bc("outflow")] * 4
    for s in range(4):
        p.bc[s] = bcs[s]
    return p


def set_shields(p: SiltProblem, formula: str = "mpm", friction: str = "manning",
                friction_coef: float | None = None, tau_cr: float = 0.047,
                grain_diameter: float = 1e-3, rel_density: float = 2.65) -> SiltProblem:
    """Switch a problem to BedloadLaw::shields (reference src/bedload.cpp:38-57).

    Defaults follow the reference's config layer (src/config.cpp:226-247):
    Manning friction; coefficient 0.025 for Manning, 0.03 for Darcy-Weisbach.
    """
    p.law_kind = LAW_SHIELDS
    p.shields_formula = SHIELDS_FORMULAS[formula]
    p.friction_model = FRICTION_MODELS[friction]
    if friction_coef is None:
        friction_coef = 0.025 if friction == "manning" else 0.03
    p.friction_coef = float(friction_coef)
    p.tau_cr = float(tau_cr)
    p.grain_diameter = float(grain_diameter)
    p.rel_density = float(rel_density)
    return p


INF = math.inf
