"""CPU: the C-ABI library builds, loads, exports every declared symbol, and its
ctypes mirror matches the C struct layout.  Argument validation that happens
before any device work is exercised here too (no GPU needed)."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1307_0491_b200 import abi, build


@pytest.fixture(scope="module")
def native():
    build.build()
    from paper_1307_0491_b200 import native as N
    return N


def declared_symbols():
    with open(os.path.join(ROOT, "include", "silt_cuda.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(silt_\w+)\s*\(", text, re.M)))


def test_exports_every_declared_symbol(native):
    lib = native.lib()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n


def test_abi_version_and_struct_sizes(native):
    lib = native.lib()
    assert lib.silt_abi_version() == abi.SILT_ABI_VERSION
    sizes = (C.c_int64 * 6)()
    lib.silt_abi_sizes(sizes, 6)
    mirror = [C.sizeof(t) for t in (abi.SiltBC, abi.SiltProblem, abi.SiltStrip,
                                    abi.SiltRunPlan, abi.SiltStatus, abi.SiltExchange)]
    assert list(sizes) == mirror


def test_validation_without_device(native):
    f = np.ones((4, 4, 4))
    p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=0.1, cfl=0.0)
    with pytest.raises(native.InvalidArgument, match="cfl"):
        native.run(p, f)
    p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=0.1, m_g=5.0)
    with pytest.raises(native.InvalidArgument, match="m_g"):
        native.Solver(p)
    p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=-1.0)
    with pytest.raises(native.InvalidArgument, match="a_g"):
        native.Solver(p)
    p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=0.1,
                         bcs=[abi.bc("periodic"), abi.bc("outflow"), abi.bc("outflow"),
                              abi.bc("outflow")])
    with pytest.raises(native.InvalidArgument, match="periodic"):
        native.Solver(p)
    p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=0.1)
    p.law_kind = 2
    with pytest.raises(native.InvalidArgument, match="law kind"):
        native.Solver(p)
    p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=0.1)
    bad = abi.SiltStrip(0, 9, 0, 0)
    with pytest.raises(native.InvalidArgument, match="partition"):
        native.Solver(p, bad)


def test_product_does_not_import_oracle():
    """The product package never loads the checkers (oracle/)."""
    pkg = os.path.join(ROOT, "paper_1307_0491_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".hpp")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "import oracle" not in src and "libsilt_oracle" not in src, f
                assert "libsilt_ref" not in src, f
