"""Shared test configuration.

Markers:
  gpu  — needs a B200 (run with `pytest -m gpu` on the GPU box); everything
         else runs on CPU in the build container.
Golden fixtures (tests/golden/) come from the reference itself
(tests/golden/make_golden.py); the oracle/ checkers are built on demand.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def _have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        meta = json.load(fh)
    return data, meta


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle as O
    if not os.path.exists(O.RESTATEMENT_SO):
        O.build(reference=False)
    return O


@pytest.fixture(scope="session")
def restatement(oracle_mod):
    return oracle_mod.restatement()


def problem_from_meta(case: dict):
    from paper_1307_0491_b200 import abi
    p = abi.make_problem(case["dim"], case["nx"], case["ny"], case["dx"], case["dy"],
                         a_g=case["a_g"], m_g=case["m_g"], cfl=case["cfl"],
                         safety=case["safety"])
    for s, (t, sup, q0, h0) in enumerate(case["bc"]):
        p.bc[s] = abi.SiltBC(t, sup, q0, h0)
    if "law" in case:  # Shields fixtures (tests/golden/make_golden_shields.py)
        abi.set_shields(p, **case["law"])
    return p


@pytest.fixture(scope="session")
def golden_shields():
    data = np.load(os.path.join(GOLDEN_DIR, "golden_shields.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden_shields.json")) as fh:
        meta = json.load(fh)
    return data, meta


def normwise(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Per-field ||a-b||_inf / ||b||_inf over the last axis."""
    a = a.reshape(-1, a.shape[-1])
    b = b.reshape(-1, b.shape[-1])
    den = np.max(np.abs(b), axis=0)
    den = np.where(den == 0, 1.0, den)
    return np.max(np.abs(a - b), axis=0) / den


def momentum_normwise(a: np.ndarray, b: np.ndarray) -> float:
    """||a_hv - b_hv||_inf / ||(hu, hv)_b||_inf: hv measured against the
    momentum vector's magnitude.  Early in a run hv is nearly zero while its
    rounding floor is set by the O(|hu|^2/h + g h^2/2) fluxes it is the
    difference of, so the per-field hv ratio measures rounding, not error
    (DESIGN.md §4)."""
    a = a.reshape(-1, a.shape[-1])
    b = b.reshape(-1, b.shape[-1])
    den = max(np.abs(b[:, 1]).max(), np.abs(b[:, 2]).max())
    return float(np.abs(a[:, 2] - b[:, 2]).max() / den)
