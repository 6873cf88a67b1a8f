"""CPU, multi-process: the row-strip driver (paper_1307_0491_b200.distributed)
over torch.distributed/gloo with world sizes 2 and 3.

Each rank steps its strip with a CPU stand-in (tests/strip_oracle.py) built on
the oracle restatement, so what is tested is the product's multi-rank host
logic: block_range partition, neighbour order (incl. the periodic G=2 case
where south == north), ghost-row send/recv pairing, the MAX all-reduce that
yields global_dt, snapshot pauses and the gather.  The reference's contract
(tests/test_parallel.cpp:215-238): every layout equals run_serial bit for bit.
"""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT
from paper_1307_0491_b200 import abi, scenarios
from paper_1307_0491_b200.distributed import block_range, neighbours


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_block_range_matches_reference_partition():
    # parallel.cpp:25-30: counts differ by <= 1, remainder to the lowest ranks
    for n, parts in ((10, 3), (16384, 8), (7, 7), (1000, 6)):
        offs, cnts = zip(*(block_range(n, parts, r) for r in range(parts)))
        assert sum(cnts) == n and max(cnts) - min(cnts) <= 1
        assert list(offs) == [sum(cnts[:r]) for r in range(parts)]
        assert sorted(cnts, reverse=True) == list(cnts)


def test_neighbours():
    assert neighbours(0, 1, False) == (None, None)
    assert neighbours(0, 1, True) == (None, None)  # one strip wraps by itself
    assert neighbours(0, 3, False) == (None, 1)
    assert neighbours(2, 3, False) == (1, None)
    assert neighbours(0, 3, True) == (2, 1)
    assert neighbours(1, 2, True) == (0, 0)


def _worker(rank, world, port, case, out_dir, partition=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_1307_0491_b200.distributed import StripRunner, init_dist
    from strip_oracle import StripOracle
    p, init, steps, snaps, bcs = case
    for s in range(4):
        p.bc[s] = bcs[s]
    init_dist(world, backend="gloo")
    orc = O.restatement()

    def factory(problem, strip):
        return StripOracle(problem, strip, orc, init[strip.j0:strip.j0 + strip.ny_local])

    runner = StripRunner(p, world, rank, solver_factory=factory, partition=partition)
    runner.begin(max_steps=steps, snapshots=snaps)
    seen = []
    st = runner.run(batch=3, on_snapshot=lambda t, f: seen.append(t))
    field = runner.gather()
    if rank == 0:
        np.save(os.path.join(out_dir, "field.npy"), field)
        np.save(os.path.join(out_dir, "meta.npy"), np.array([st.t, st.steps] + seen))
    runner.shutdown()


CASES = {
    "random_outflow": (lambda: scenarios.random_bed_2d(24, 13, a_g=0.3), 12, (),
                       [abi.bc("outflow")] * 4),
    "periodic_y": (lambda: scenarios.random_bed_2d(20, 12, a_g=0.3), 10, (0.7,),
                   [abi.bc("inflow", q0=1.0), abi.bc("wall"), abi.bc("periodic"),
                    abi.bc("periodic")]),
    "walls": (lambda: scenarios.random_bed_2d(18, 11, a_g=0.2), 10, (0.4, 0.9),
              [abi.bc("wall"), abi.bc("outflow"), abi.bc("wall"),
               abi.bc("inflow", q0=-0.5)]),
}


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", sorted(CASES))
def test_strips_bitwise_equal_serial(tmp_path, restatement, world, case):
    build, steps, snaps, bcs = CASES[case]
    p, init, _ = build()
    for s in range(4):
        p.bc[s] = bcs[s]
    ref, t, n, _ = restatement.run(p, init, max_steps=steps, snapshots=snaps)
    mp.spawn(_worker, args=(world, _free_port(), (p, init, steps, snaps, bcs), str(tmp_path)),
             nprocs=world, join=True)
    field = np.load(tmp_path / "field.npy")
    meta = np.load(tmp_path / "meta.npy")
    assert meta[1] == n and meta[0] == t
    assert list(meta[2:]) == [s for s in snaps if s <= t]
    assert np.array_equal(field, ref)


def test_uneven_partition_bitwise_equal_serial(tmp_path, restatement):
    """Work-balanced (uneven) strips: any partition gives the serial result."""
    from paper_1307_0491_b200.distributed import balanced_partition, row_costs
    p, init, _ = scenarios.dune_2d(32, a_g=0.5)
    steps = 12
    part = balanced_partition(row_costs(init, halo=2), 3)
    assert len({n for _, n in part}) > 1  # genuinely uneven
    ref, t, n, _ = restatement.run(p, init, max_steps=steps)
    bcs = [p.bc[s] for s in range(4)]
    mp.spawn(_worker, args=(3, _free_port(), (p, init, steps, (), bcs), str(tmp_path), part),
             nprocs=3, join=True)
    assert np.array_equal(np.load(tmp_path / "field.npy"), ref)


def test_balanced_partition_properties():
    from paper_1307_0491_b200.distributed import balanced_partition
    rng = np.random.default_rng(3)
    for n, parts in ((100, 7), (16384, 8), (9, 9)):
        cost = rng.uniform(0.1, 5.0, n)
        part = balanced_partition(cost, parts)
        assert part[0][0] == 0 and sum(c for _, c in part) == n
        assert all(c >= 1 for _, c in part)
        assert all(part[k][0] + part[k][1] == part[k + 1][0] for k in range(parts - 1))
        if n > 1000:
            loads = [cost[o:o + c].sum() for o, c in part]
            assert max(loads) <= 1.01 * sum(loads) / parts


def test_piece_partition_layout():
    """Two pieces per rank (distributed.piece_partition): the 2N pieces tile
    the rows exactly once, the hot pieces cover the mound's rows, and no two
    pieces of one rank are row neighbours (their exchange is always between
    processes)."""
    from paper_1307_0491_b200 import scenarios
    from paper_1307_0491_b200.distributed import piece_order, piece_partition, row_costs
    p, init, _ = scenarios.dune_2d(1024)
    costs = row_costs(init)
    hot_rows = np.nonzero(costs > costs.min() * (1 + 1e-9))[0]
    for world in (2, 3, 4, 5, 8):
        layout = piece_partition(costs, world)
        assert len(layout) == world and all(len(x) == 2 for x in layout)
        order = piece_order(layout)
        assert order[0][0] == 0 and sum(n for _, n, _, _ in order) == 1024
        assert all(a[0] + a[1] == b[0] for a, b in zip(order, order[1:]))
        assert all(a[2] != b[2] for a, b in zip(order, order[1:]))
        hot = [x[0] for x in layout]
        lo, hi = min(j for j, _ in hot), max(j + n for j, n in hot)
        assert lo <= hot_rows[0] and hi > hot_rows[-1]
    # a grid without a distinct hot band keeps contiguous strips
    flat = np.ones(1024)
    assert piece_partition(flat, 4) is None
