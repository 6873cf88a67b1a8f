"""Host-side input generation for the BASELINE configurations C1-C5.

Initial data are built on the host once and fed identically to the oracle and
to the GPU path.  C1-C4 follow the analytic profiles of BASELINE.json and use
``math.sin`` element by element (the same libm ``sin`` the reference's
``sine_bump`` calls, src/scenarios.cpp:146-149 / 255-287) so the arrays match the
reference's own builders bit for bit.  C5 (random bed) has no reference
generator; ours is documented in DESIGN.md §Inputs: a counter-based
(splitmix64) uniform/normal stream, a periodic Gaussian filter of sigma = 20
cells applied by FFT, normalisation to unit variance, clipping to [-1, 1].

Every builder returns (problem, init, steps) where init is a float64 array of
shape (ny, nx, 4) holding FlowState {h, hu, hv, zb} (reference
include/silt/grid.hpp:44-49, row-major, i fastest).
"""
from __future__ import annotations

import math

import numpy as np

from .abi import SiltProblem, bc, make_problem


def _sine_bump(x: np.ndarray, start: float, width: float) -> np.ndarray:
    """sine_bump (src/scenarios.cpp:146-149) on [start, start+width], else 0."""
    out = np.zeros_like(x)
    for k, xv in enumerate(x.tolist()):
        if start <= xv <= start + width:
            s = math.sin((xv - start) * math.pi / width)
            out[k] = s * s
    return out


def _centres(n: int, d: float) -> np.ndarray:
    """Grid::x_center (include/silt/grid.hpp:35-36): (i + 1/2) dx."""
    return (np.arange(n, dtype=np.float64) + 0.5) * d


def dune_1d(cells: int = 1000, a_g: float = 1.0, cfl: float = 0.5,
            steps: int = 1000):
    """C1: 1D dune, [0,1000] m, zb=0.1+sin^2 on [300,500], h=10-zb, hu=10."""
    dx = 1000.0 / cells
    x = _centres(cells, dx)
    zb = 0.1 + _sine_bump(x, 300.0, 200.0)
    init = np.zeros((1, cells, 4))
    init[0, :, 0] = 10.0 - zb
    init[0, :, 1] = 10.0
    init[0, :, 3] = zb
    p = make_problem(1, cells, 1, dx, 1.0, a_g=a_g, cfl=cfl)
    return p, init, steps


def antidune_1d(cells: int = 4000, a_g: float = 0.005, cfl: float = 0.45,
                steps: int = 5000):
    """C2: supercritical 1D, zb=0.05+0.05 sin^2 on [300,500], h=0.5-zb, hu=2.5."""
    dx = 1000.0 / cells
    x = _centres(cells, dx)
    zb = 0.05 + 0.05 * _sine_bump(x, 300.0, 200.0)
    init = np.zeros((1, cells, 4))
    init[0, :, 0] = 0.5 - zb
    init[0, :, 1] = 2.5
    init[0, :, 3] = zb
    p = make_problem(1, cells, 1, dx, 1.0, a_g=a_g, cfl=cfl)
    return p, init, steps


def dune_2d(n: int = 1024, a_g: float = 0.001, cfl: float = 0.5,
            steps: int = 1000, ny: int | None = None):
    """C3 (n=1024) / C4 (n=16384): [0,1000]^2 m, mound on [300,500]x[400,600],
    zb = 0.1 + wx*wy, h = 10 - zb, hu = 10, hv = 0 (cf. build_bump_2d,
    src/scenarios.cpp:255-287, with transmissive boundaries on every side)."""
    ny = n if ny is None else ny
    dx = 1000.0 / n
    dy = 1000.0 / ny
    wx = _sine_bump(_centres(n, dx), 300.0, 200.0)
    wy = _sine_bump(_centres(ny, dy), 400.0, 200.0)
    init = np.zeros((ny, n, 4))
    zb = 0.1 + np.multiply.outer(wy, wx)
    init[:, :, 0] = 10.0 - zb
    init[:, :, 1] = 10.0
    init[:, :, 3] = zb
    p = make_problem(2, n, ny, dx, dy, a_g=a_g, cfl=cfl)
    return p, init, steps


def _splitmix64(idx: np.ndarray, seed: int) -> np.ndarray:
    z = (idx.astype(np.uint64) + np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
         + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _uniform(n: int, seed: int, stream: int) -> np.ndarray:
    """Counter-based U[0,1) doubles: 53 high bits of splitmix64(counter)."""
    with np.errstate(over="ignore"):
        bits = _splitmix64(np.arange(n, dtype=np.uint64) + np.uint64(stream << 40), seed)
    return (bits >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def random_bed_2d(nx: int = 8192, ny: int = 32768, a_g: float = 0.01,
                  cfl: float = 0.4, steps: int = 300, seed: int = 1307,
                  sigma: float = 20.0, d: float = 1.0):
    """C5: random-bed stress test (BASELINE.json configs[4]).

    zb = 0.1 + 0.05 clip(GRF, -1, 1) with GRF = Gaussian filter (sigma cells,
    periodic, FFT) of a seeded N(0,1) field normalised to unit variance;
    h = 2 - zb; hu ~ U(0.5, 1.5); hv ~ U(-0.1, 0.1); dx = dy = d = 1 m.
    """
    n = nx * ny
    u1 = _uniform(n, seed, 0)
    u2 = _uniform(n, seed, 1)
    normal = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
    normal = normal.reshape(ny, nx)
    kx = np.fft.rfftfreq(nx)
    ky = np.fft.fftfreq(ny)
    filt = np.exp(-2.0 * (np.pi * sigma) ** 2 * (ky[:, None] ** 2 + kx[None, :] ** 2))
    grf = np.fft.irfft2(np.fft.rfft2(normal) * filt, s=(ny, nx))
    grf = (grf - grf.mean()) / grf.std()
    zb = 0.1 + 0.05 * np.clip(grf, -1.0, 1.0)
    init = np.zeros((ny, nx, 4))
    init[:, :, 0] = 2.0 - zb
    init[:, :, 1] = 0.5 + _uniform(n, seed, 2).reshape(ny, nx)
    init[:, :, 2] = -0.1 + 0.2 * _uniform(n, seed, 3).reshape(ny, nx)
    init[:, :, 3] = zb
    p = make_problem(2, nx, ny, d, d, a_g=a_g, cfl=cfl)
    return p, init, steps


CONFIGS = {
    "C1": lambda: dune_1d(),
    "C2": lambda: antidune_1d(),
    "C3": lambda: dune_2d(1024, steps=1000),
    "C4": lambda: dune_2d(16384, steps=500),
    "C5": lambda: random_bed_2d(),
}
