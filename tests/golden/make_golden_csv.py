"""Write a snapshot CSV fixture with the REFERENCE's snapshot_to_string
(src/snapshot.cpp:50-84), for the CSV parity tests (tests/test_snapshot_csv.py).

    make -C oracle && python tests/golden/make_golden_csv.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from conftest import problem_from_meta  # noqa: E402


def main() -> None:
    data = np.load(os.path.join(HERE, "golden.npz"))
    meta = json.load(open(os.path.join(HERE, "golden.json")))
    m = meta["cases"]["rand48x32"]
    p = problem_from_meta(m)
    csv = O.reference().snapshot_to_string(p, data["rand48x32_final"], m["t_final"])
    with open(os.path.join(HERE, "snapshot_rand48x32.csv"), "wb") as fh:
        fh.write(csv)
    print(len(csv), "bytes")


if __name__ == "__main__":
    main()
