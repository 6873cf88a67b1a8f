"""GPU, multi-process: the row-strip driver (StripRunner) with the real CUDA
solver in every rank, on one B200.

With SILT_P2P unset (default) the ranks exchange over peer memory (CUDA IPC:
the step kernels store edge rows into the neighbours' buffers, maxima by
remote atomics, stream memory operations order the steps); SILT_P2P=0 runs
the collective path (here gloo, host-staged; NCCL on the multi-GPU box).

The round-end and SCALE runs use StripRunner over NCCL with one GPU per rank;
a gpurun box has one GPU and NCCL refuses two ranks on one device, so these
ranks talk over gloo (edge rows and the speed slot staged through host
memory) while everything on the device side is the production path: the step
kernels writing the send rows and the reduction slot, the ghost rows read
from the receive buffers, the MAX-reduced slot driving the next launch's dt,
snapshot pauses and the gather.  No kernel waits on another rank (all
synchronisation is host-side), so sharing the GPU is safe.  The bar is the
reference's layout contract (tests/test_parallel.cpp:215-238): STRICT strips
equal the single-domain reference run bit for bit.
"""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT, normwise, problem_from_meta

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_dir, variant, partition):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    from conftest import problem_from_meta
    from paper_1307_0491_b200.distributed import StripRunner, init_dist
    m, init = case
    p = problem_from_meta(m)
    torch.cuda.set_device(0)
    init_dist(world, backend="gloo")
    runner = StripRunner(p, world, rank, device=0, variant=variant, partition=partition)
    runner.upload_host(np.ascontiguousarray(init[runner.j0:runner.j0 + runner.nrows]))
    runner.begin(max_steps=m["max_steps"], snapshots=m["snapshots"])
    seen = []
    st = runner.run(batch=4, on_snapshot=lambda t, f: seen.append(t))
    field = runner.gather()
    if rank == 0:
        np.save(os.path.join(out_dir, "field.npy"), field)
        np.save(os.path.join(out_dir, "meta.npy"), np.array([st.t, st.steps] + seen))
        np.save(os.path.join(out_dir, "mode.npy"), np.array([runner._p2p, runner._overlap]))
    runner.close()
    runner.shutdown()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["rand48x32", "bc_periodic", "bc_inflow_wall"])
def test_strip_runner_ranks_on_one_gpu(tmp_path, golden, world, case):
    import torch.multiprocessing as mp
    from paper_1307_0491_b200 import abi
    data, meta = golden
    m = meta["cases"][case]
    init = data[f"{case}_init"]
    for variant, part in ((abi.VARIANT_STRICT, None), (abi.VARIANT_FAST, None)):
        out = tmp_path / f"v{variant}"
        out.mkdir()
        mp.spawn(_worker, args=(world, _free_port(), (m, init), str(out), variant, part),
                 nprocs=world, join=True)
        field = np.load(out / "field.npy")
        mt = np.load(out / "meta.npy")
        p2p, _ = np.load(out / "mode.npy")
        assert bool(p2p) == (os.environ.get("SILT_P2P", "1") != "0")  # the path under test
        assert mt[1] == m["steps"]
        assert list(mt[2:]) == [s for s in m["snapshots"] if s <= m["t_final"]]
        if variant == abi.VARIANT_STRICT:
            assert mt[0] == m["t_final"]
            assert np.array_equal(field, data[f"{case}_final"])
        else:
            assert np.all(normwise(field, data[f"{case}_final"]) <= 1e-9)


def _piece_worker(rank, world, port, n, steps, out_dir, variant):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    sys.path.insert(0, ROOT)
    import torch
    from paper_1307_0491_b200 import scenarios
    from paper_1307_0491_b200.distributed import PieceRunner, init_dist, piece_partition, row_costs
    p, init, _ = scenarios.dune_2d(n)
    torch.cuda.set_device(0)
    init_dist(world, backend="gloo")
    layout = piece_partition(row_costs(init), world)
    runner = PieceRunner(p, world, rank, layout, device=0, variant=variant)
    runner.upload_host(init)
    runner.begin(max_steps=steps, dt_cap=steps)
    runner.step(steps)
    runner.synchronize()
    st = runner.status()
    field = runner.gather()
    if rank == 0:
        np.save(os.path.join(out_dir, "field.npy"), field)
        np.save(os.path.join(out_dir, "meta.npy"), np.array([st.t, st.steps]))
        np.save(os.path.join(out_dir, "dt.npy"), runner.dt_log(steps))
        with open(os.path.join(out_dir, "layout.txt"), "w") as fh:
            fh.write(repr(layout))
    runner.close()
    runner.shutdown()


@pytest.mark.parametrize("world", [2, 3])
def test_two_pieces_per_rank_on_one_gpu(tmp_path, restatement, world):
    """PieceRunner (two row ranges per rank — 1/N of the hot band around the
    mound + 1/N of the far field — stepped concurrently, peer-memory exchange
    between all 2N pieces): bitwise equal to the reference's serial run
    (STRICT), FAST within the bar."""
    import torch.multiprocessing as mp
    from paper_1307_0491_b200 import abi, scenarios
    if os.environ.get("SILT_P2P", "1") == "0":
        pytest.skip("peer-memory path disabled")
    n, steps = 160, 30
    p, init, _ = scenarios.dune_2d(n)
    ref, t, sn, log = restatement.run(p, init, max_steps=steps)
    for variant in (abi.VARIANT_STRICT, abi.VARIANT_FAST):
        out = tmp_path / f"v{variant}"
        out.mkdir()
        mp.spawn(_piece_worker, args=(world, _free_port(), n, steps, str(out), variant),
                 nprocs=world, join=True)
        field = np.load(out / "field.npy")
        t_got, steps_got = np.load(out / "meta.npy")
        assert steps_got == sn
        if variant == abi.VARIANT_STRICT:
            assert t_got == t
            assert np.array_equal(np.load(out / "dt.npy"), log)
            assert np.array_equal(field, ref), (out / "layout.txt").read_text()
        else:
            assert np.all(normwise(field, ref) <= 1e-9)


def _hung_peer_worker(rank, world, port, case, out_dir):
    """Rank 1 stops stepping after begin (a hung or dying peer); rank 0's
    bounded peer wait must turn that into an error instead of spinning."""
    import time
    os.environ["SILT_P2P_TIMEOUT_MS"] = "2000"
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    from conftest import problem_from_meta
    from paper_1307_0491_b200 import abi, native
    from paper_1307_0491_b200.distributed import StripRunner, init_dist
    m, init = case
    p = problem_from_meta(m)
    torch.cuda.set_device(0)
    init_dist(world, backend="gloo")
    runner = StripRunner(p, world, rank, device=0, variant=abi.VARIANT_FAST)
    runner.upload_host(np.ascontiguousarray(init[runner.j0:runner.j0 + runner.nrows]))
    runner.begin(max_steps=m["max_steps"])
    done = os.path.join(out_dir, "result.txt")
    if rank == 1:  # hung: never steps; keeps its memory mapped until rank 0 is done
        t0 = time.time()
        while not os.path.exists(done) and time.time() - t0 < 120:
            time.sleep(0.2)
        os._exit(0)
    msg = "no error"
    t0 = time.time()
    try:
        runner.step(4)
        runner.status()
    except native.SiltRuntimeError as e:
        msg = str(e)
    el = time.time() - t0
    with open(done + ".tmp", "w") as fh:
        fh.write(f"{runner._p2p}\n{el}\n{msg}\n")
    os.replace(done + ".tmp", done)
    os._exit(0)


def test_hung_peer_times_out(tmp_path, golden):
    """Peer-memory strips: a rank that stops publishing its steps makes the
    others fail with an error naming it (bounded wait in the acquire kernel,
    SILT_P2P_TIMEOUT_MS) instead of hanging the GPU."""
    import torch.multiprocessing as mp
    if os.environ.get("SILT_P2P", "1") == "0":
        pytest.skip("peer-memory path disabled")
    data, meta = golden
    m = meta["cases"]["rand48x32"]
    mp.spawn(_hung_peer_worker, args=(2, _free_port(), (m, data["rand48x32_init"]),
                                      str(tmp_path)), nprocs=2, join=True)
    p2p, el, msg = (tmp_path / "result.txt").read_text().splitlines()[:3]
    assert p2p == "True"
    assert "rank 1 did not publish step 1" in msg, msg
    assert float(el) < 30.0


def test_uneven_partition_on_one_gpu(tmp_path, golden):
    """A work-balanced (uneven) partition through the same device path."""
    import torch.multiprocessing as mp
    from paper_1307_0491_b200 import abi
    data, meta = golden
    m = meta["cases"]["dune64_ag1"]
    part = [(0, 13), (13, 40), (53, 11)]
    mp.spawn(_worker, args=(3, _free_port(), (m, data["dune64_ag1_init"]), str(tmp_path),
                            abi.VARIANT_STRICT, part), nprocs=3, join=True)
    assert np.array_equal(np.load(tmp_path / "field.npy"), data["dune64_ag1_final"])


def test_bench_two_ranks_on_one_gpu():
    """bench.py's N > 1 path (torchrun, the two-pieces-per-rank layout forced
    down to N = 2, max-over-ranks timing, e2e) end to end, two ranks sharing
    the GPU over gloo: one valid JSON line from rank 0."""
    import json
    import subprocess
    env = dict(os.environ, SILT_DIST_BACKEND="gloo", SILT_PIECES_MIN="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "C3", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["layout"]["parallelism"] == "row strips x2"
    assert d["layout"]["partition"].startswith("two pieces per rank")
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
