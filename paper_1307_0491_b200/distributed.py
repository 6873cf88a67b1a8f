"""Row-strip domain decomposition across GPUs (one process per GPU).

The reference runs the paper's MPI decomposition as SPMD threads
(run_parallel, src/parallel.cpp:261-386): Cartesian blocks (partition,
:150-177), a one-cell pull halo (pull_halo, :43-84) and an exact-min global dt
(global_dt, :200-206).  Here every rank owns a strip of whole rows
(Topology{px=1, py=G}, remainder rows to the lowest ranks as in block_range,
:25-30) resident in its GPU's HBM.  Per step, in stream order and with no host
synchronisation:

  1. the fused step kernel advances the strip and writes its edge rows into
     send buffers plus its CFL speed maxima into the reduction slot;
  2. ghost rows move to the neighbours (NCCL send/recv: ``batch_isend_irecv``);
  3. the two axis-speed maxima are all-reduced with MAX (16 bytes).  Because
     correctly rounded division is monotone, min over ranks of
     cfl*min(dx/sx_r, dy/sy_r) == cfl*min(dx/max sx, dy/max sy): the dt every
     rank derives on device equals global_dt bit for bit.

``depth hmax`` stays per strip (the reference's per-worker check_depth).
The same driver runs on CPU with the gloo backend for the tests, with any
object that implements the strip-solver interface below.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi


def block_range(n: int, parts: int, r: int):
    """block_range (src/parallel.cpp:25-30): (offset, count)."""
    base, rem = divmod(n, parts)
    count = base + (1 if r < rem else 0)
    offset = r * base + min(r, rem)
    return offset, count


def neighbours(rank: int, world: int, periodic_y: bool):
    """Topology::neighbor (src/parallel.cpp:136-148) for px = 1, py = world:
    (south rank or None, north rank or None)."""
    south = rank - 1 if rank > 0 else (world - 1 if periodic_y and world > 1 else None)
    north = rank + 1 if rank < world - 1 else (0 if periodic_y and world > 1 else None)
    return south, north


def balanced_partition(row_cost, parts: int):
    """Row strips of (approximately) equal total cost: returns [(offset,
    count)] with every count >= 1.  Any partition gives bit-identical results
    (the reference's layout contract, tests/test_parallel.cpp:215-238), so the
    strips may follow the work instead of block_range's equal row counts."""
    cost = np.asarray(row_cost, dtype=np.float64)
    n = cost.size
    if parts < 1 or parts > n:
        raise ValueError("partition: every worker needs at least one cell per axis")
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    cuts = [0]
    for k in range(1, parts):
        target = cum[-1] * k / parts
        c = int(np.searchsorted(cum, target))
        c = max(c, cuts[-1] + 1)            # >= 1 row per strip
        c = min(c, n - (parts - k))         # leave >= 1 row for each later strip
        cuts.append(c)
    cuts.append(n)
    return [(cuts[k], cuts[k + 1] - cuts[k]) for k in range(parts)]


QUIET_COST = 1.0 / 10.0  # measured on C4 strips (tools/strip_times.py): quiescent vs active segment


def row_costs(field, h_dry: float = 1e-8, seg: int = 30, halo: int = 32):
    """Estimated step cost per row of a (ny, nx, 4) field (numpy or torch):
    30-cell segments whose cells equal their x and y neighbours are quiescent
    (the step kernel skips them), the rest pay the full Riemann solves.  The
    active set is dilated by ``halo`` rows to cover waves spreading during the
    run."""
    try:
        import torch
        is_t = isinstance(field, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_t = False
    if is_t:
        f = field
        same_x = (f[:, 1:] == f[:, :-1]).all(dim=-1)
        same_y = (f[1:] == f[:-1]).all(dim=-1)
        q = torch.ones(f.shape[:2], dtype=torch.bool, device=f.device)
        q[:, 1:] &= same_x
        q[:, :-1] &= same_x
        q[1:] &= same_y
        q[:-1] &= same_y
        q &= f[..., 0] > h_dry
        q = q.cpu().numpy()
    else:
        f = np.asarray(field)
        same_x = (f[:, 1:] == f[:, :-1]).all(axis=-1)
        same_y = (f[1:] == f[:-1]).all(axis=-1)
        q = np.ones(f.shape[:2], dtype=bool)
        q[:, 1:] &= same_x
        q[:, :-1] &= same_x
        q[1:] &= same_y
        q[:-1] &= same_y
        q &= f[..., 0] > h_dry
    ny, nx = q.shape
    nseg = (nx + seg - 1) // seg
    pad = np.ones((ny, nseg * seg), dtype=bool)
    pad[:, :nx] = q
    seg_quiet = pad.reshape(ny, nseg, seg).all(axis=2)
    active = ~seg_quiet
    if halo > 0:  # dilate along y
        act = active.copy()
        for d in range(1, halo + 1):
            act[d:] |= active[:-d]
            act[:-d] |= active[d:]
        active = act
    return active.sum(axis=1) + QUIET_COST * (~active).sum(axis=1)


def refine_partition(row_cost, partition, strip_ms):
    """One measured refinement: rescale the modelled cost of every row by its
    strip's measured/predicted time, then re-cut.  strip_ms[k] is the measured
    step time of partition[k]."""
    cost = np.asarray(row_cost, dtype=np.float64).copy()
    for (j0, n), t in zip(partition, strip_ms):
        pred = cost[j0:j0 + n].sum()
        if pred > 0 and t > 0:
            cost[j0:j0 + n] *= t / pred
    return balanced_partition(cost, len(partition))


def init_dist(gpus: int = 1, backend: str | None = None):
    """(world, rank, local_rank); initialises torch.distributed when world > 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            if backend is None:  # SILT_DIST_BACKEND=gloo: multi-rank tests on one GPU
                backend = os.environ.get("SILT_DIST_BACKEND") or (
                    "nccl" if torch.cuda.is_available() else "gloo")
            kw = {}
            if backend == "nccl":
                kw["device_id"] = torch.device("cuda", local)
            dist.init_process_group(backend, **kw)
    return world, rank, local


class _CAI:
    """Zero-copy view of a device buffer for torch (CUDA array interface)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class StripRunner:
    """One rank's strip: a solver + the per-step halo/dt exchange.

    ``solver`` defaults to the CUDA solver (native.Solver) on ``device``; tests
    pass a CPU stand-in with the same interface.
    """

    def __init__(self, problem, world: int, rank: int, device: int = 0,
                 variant: int = abi.VARIANT_FAST, solver_factory=None, partition=None):
        self.problem = problem
        self.world, self.rank = world, rank
        ny = 1 if problem.dim == 1 else problem.ny
        if world > ny:
            raise ValueError("partition: every worker needs at least one cell per axis")
        if problem.dim == 1 and world > 1:
            raise ValueError("partition: 1D grids require py == 1")
        if partition is None:  # block_range, the reference's partition
            self.j0, self.nrows = block_range(ny, world, rank)
        else:  # e.g. balanced_partition(row_costs(...), world): [(j0, n)] per rank
            if len(partition) != world or sum(n for _, n in partition) != ny:
                raise ValueError("partition: strips must cover the grid once")
            self.j0, self.nrows = partition[rank]
        periodic_y = problem.dim == 2 and problem.bc[abi.SOUTH].type == abi.BC_PERIODIC
        self.south, self.north = neighbours(rank, world, periodic_y)
        strip = abi.SiltStrip(self.j0, self.nrows, int(self.south is not None),
                              int(self.north is not None))
        self.torch_stream = None
        if solver_factory is None:
            import torch
            from . import native
            self.solver = native.Solver(problem, strip, device, variant)
            self.torch_stream = torch.cuda.Stream(device=device)
            self.solver.set_stream(self.torch_stream.cuda_stream)
            self.device = torch.device("cuda", device)
            ex = self.solver.exchange_ptrs()
            n = ex.row_doubles
            self._send_s = self._wrap(ex.send_south, n)
            self._send_n = self._wrap(ex.send_north, n)
            self._recv_s = self._wrap(ex.recv_south, n)
            self._recv_n = self._wrap(ex.recv_north, n)
        else:
            self.solver = solver_factory(problem, strip)
            self.device = None
            self._send_s, self._send_n, self._recv_s, self._recv_n = self.solver.exchange_tensors()
        self._dist = None
        self._stage = False
        if world > 1:
            import torch.distributed as dist
            self._dist = dist
            # gloo moves CPU tensors only: device rows are staged through host
            # memory (used by the one-GPU multi-process tests; NCCL moves the
            # device buffers directly)
            self._stage = self.torch_stream is not None and dist.get_backend() == "gloo"
        # Peer-memory exchange (silt_solver_p2p_*): the step kernels deliver
        # the edge rows into the neighbours' memory and the maxima by remote
        # atomics, ordered by stream memory operations — no collective per
        # step.  Every rank must succeed, else all use the collective path.
        # SILT_P2P=0 disables.
        self._p2p = False
        if (world > 1 and self.torch_stream is not None and problem.dim == 2 and
                os.environ.get("SILT_P2P", "1") != "0"):
            self._p2p = self._setup_p2p()
        # halo/compute overlap (silt_solver_step_part); SILT_OVERLAP=0 disables
        self._overlap = (not self._p2p and world > 1 and self.torch_stream is not None and
                         os.environ.get("SILT_OVERLAP", "1") != "0" and self.solver.split_ok())
        if self._overlap and not self._stage:
            import torch
            self._comm = torch.cuda.Stream(device=self.device)
            self._ev = torch.cuda.Event()

    def _setup_p2p(self) -> bool:
        import torch
        dist = self._dist
        ok = 1
        handle = b""
        try:
            handle = self.solver.p2p_export()
        except Exception:
            ok = 0
        handles = [None] * self.world
        dist.all_gather_object(handles, handle)
        if ok and all(handles):
            try:
                self.solver.p2p_connect(self.rank, self.world, handles, self.south, self.north)
            except Exception:
                ok = 0
        else:
            ok = 0
        t = torch.tensor([ok], dtype=torch.int32,
                         device=self.device if not self._stage else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) != 1:
            if ok:  # connected here but not everywhere: not usable
                raise RuntimeError("p2p: connected on some ranks only")
            return False
        return True

    def _wrap(self, ptr, n):
        if not ptr:
            return None
        import torch
        return torch.as_tensor(_CAI(ptr, n), device=self.device)

    def _slot(self):
        if self.torch_stream is None:
            return self.solver.reduce_slot_tensor()
        import torch
        return torch.as_tensor(_CAI(self.solver.reduce_slot(), 2), device=self.device)

    # ---- exchange ---------------------------------------------------------
    def _row_ops(self, send_n, recv_s, send_s, recv_n):
        """Order per rank: send north, recv south, send south, recv north —
        consistent pairing also when south == north (periodic, G = 2)."""
        dist = self._dist
        ops = []
        if self.north is not None:
            ops.append(dist.P2POp(dist.isend, send_n, self.north))
        if self.south is not None:
            ops.append(dist.P2POp(dist.irecv, recv_s, self.south))
        if self.south is not None:
            ops.append(dist.P2POp(dist.isend, send_s, self.south))
        if self.north is not None:
            ops.append(dist.P2POp(dist.irecv, recv_n, self.north))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def _exchange_rows(self):
        """Edge rows of the newest state to the neighbours' ghost rows."""
        if not self._stage:
            self._row_ops(self._send_n, self._recv_s, self._send_s, self._recv_n)
            return
        # gloo moves host tensors: stage the device rows
        self.torch_stream.synchronize()
        sn = self._send_n.cpu() if self._send_n is not None else None
        ss = self._send_s.cpu() if self._send_s is not None else None
        rs = self._recv_s.cpu() if self._recv_s is not None else None
        rn = self._recv_n.cpu() if self._recv_n is not None else None
        self._row_ops(sn, rs, ss, rn)
        with self._ctx():
            if rs is not None:
                self._recv_s.copy_(rs)
            if rn is not None:
                self._recv_n.copy_(rn)

    def _reduce_slot(self):
        """MAX of the axis speeds over all ranks (global_dt, src/parallel.cpp:200-206)."""
        dist = self._dist
        slot = self._slot()
        if not self._stage:
            dist.all_reduce(slot, op=dist.ReduceOp.MAX)
            return
        self.torch_stream.synchronize()
        s = slot.cpu()
        dist.all_reduce(s, op=dist.ReduceOp.MAX)
        with self._ctx():
            slot.copy_(s)

    def _exchange(self):
        """Ghost rows of the newest state to the neighbours, then MAX of the
        axis speeds."""
        if self.world == 1:
            return
        self._exchange_rows()
        self._reduce_slot()

    def _step_overlapped(self):
        """One step with the edge-row exchange overlapping the interior: the
        boundary row blocks first (they read the received rows and write the
        send rows), the exchange on a side stream after them, the interior
        blocks meanwhile on the solver's stream, then the MAX all-reduce."""
        import torch
        self.solver.step_part(1)
        if self._stage:  # gloo: host-staged, no concurrency, same device work
            self._exchange_rows()
            self.solver.step_part(2)
            self._reduce_slot()
            return
        self._ev.record(self.torch_stream)
        with torch.cuda.stream(self._comm):
            self._comm.wait_event(self._ev)
            self._row_ops(self._send_n, self._recv_s, self._send_s, self._recv_n)
        self.solver.step_part(2)
        self.torch_stream.wait_stream(self._comm)
        self._reduce_slot()

    def _ctx(self):
        if self.torch_stream is None:
            import contextlib
            return contextlib.nullcontext()
        import torch
        return torch.cuda.stream(self.torch_stream)

    # ---- solver interface ----------------------------------------------------
    def upload_device(self, tensor):
        # the tensor was produced on torch's current stream; the solver copies
        # on its own stream, so order the two first
        if tensor.is_cuda:
            import torch
            torch.cuda.current_stream(tensor.device).synchronize()
        self.solver.upload_device(tensor.data_ptr())
        if self.torch_stream is not None:
            self.torch_stream.synchronize()

    def upload_host(self, array):
        if hasattr(array, "data_ptr"):
            import ctypes as C
            from .native import check
            check(self.solver.L.silt_solver_upload(self.solver.h,
                                                   C.cast(array.data_ptr(), C.POINTER(C.c_double))))
        else:
            self.solver.upload(array)

    def download_host(self, out):
        if hasattr(out, "data_ptr"):
            import ctypes as C
            from .native import check
            check(self.solver.L.silt_solver_download(self.solver.h,
                                                     C.cast(out.data_ptr(), C.POINTER(C.c_double))))
            return out
        return self.solver.download(out)

    def begin(self, t_end: float = np.inf, max_steps: int = -1, snapshots=(), dt_cap: int = 0):
        with self._ctx():
            self.solver.begin(t_end=t_end, max_steps=max_steps, snapshots=snapshots,
                              dt_cap=dt_cap)
            if self._p2p:
                # the initial reduction delivered the edge rows itself; the
                # MAX all-reduce finishes global_dt and orders every rank's
                # initial kernels before any first step
                self._reduce_slot()
            else:
                self._exchange()

    def step(self, n: int = 1):
        with self._ctx():
            if self.world == 1:
                self.solver.step(n)
                return
            if self._p2p:
                self.solver.p2p_step(n)
                return
            for _ in range(n):
                if self._overlap:
                    self._step_overlapped()
                else:
                    self.solver.step(1)
                    self._exchange()

    def status(self):
        return self.solver.status()

    def resume(self):
        self.solver.resume()

    def launch_count(self) -> int:
        return self.solver.launch_count()

    def synchronize(self):
        if self.torch_stream is not None:
            self.torch_stream.synchronize()

    def record_join(self):
        """(PieceRunner interface) the solver's stream IS torch_stream."""

    def barrier(self):
        if self._dist is not None:
            self._dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        if self._dist is None:
            return v
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64,
                         device=self.device if self.device is not None else "cpu")
        self._dist.all_reduce(t, op=self._dist.ReduceOp.MAX)
        return float(t.item())

    def run(self, batch: int = 16, on_snapshot=None):
        """run_parallel's loop: advance until DONE, gathering at snapshots."""
        while True:
            self.step(batch)
            st = self.status()
            if st.state == abi.STATE_PAUSED:
                if on_snapshot is not None:
                    f = self.gather()
                    if self.rank == 0:
                        on_snapshot(st.t, f)
                self.resume()
                continue
            if st.state == abi.STATE_DONE:
                return st

    def gather(self):
        """gather (src/parallel.cpp:179-190): the global field on rank 0."""
        local = self.solver.download()
        if self.world == 1:
            return local
        parts = [None] * self.world if self.rank == 0 else None
        self._dist.gather_object(local, parts, dst=0)
        if self.rank != 0:
            return None
        return np.concatenate(parts, axis=0)

    def close(self):
        if self._p2p:
            # peers may still be storing into this rank's memory: every rank
            # drains its stream before any rank frees its buffers
            self.torch_stream.synchronize()
            self._dist.barrier()
        self.solver.close()

    def shutdown(self):
        if self._dist is not None and self._dist.is_initialized():
            self._dist.destroy_process_group()


class LocalStripGroup:
    """run_parallel(sc, 1, py) in ONE process (src/parallel.cpp:261-386): py
    row strips, strip k on CUDA device ``devices[k % len(devices)]`` — the
    native strip group of the C ABI (silt_group_*): ghost rows move with
    device/peer copies and the axis-speed maxima are reduced on device,
    ordered by stream events, so no step needs a host round trip.
    """

    def __init__(self, problem, py: int, devices=(0,), variant: int = abi.VARIANT_FAST):
        import ctypes as C
        from . import native
        self.N = native
        self.L = native.lib()
        self.problem = problem
        self.nx = problem.nx
        self.ny = 1 if problem.dim == 1 else problem.ny
        devs = (C.c_int * len(devices))(*devices)
        self.h = C.c_void_p()
        native.check(self.L.silt_group_create(C.byref(problem), int(py), devs, len(devices),
                                              variant, C.byref(self.h)))

    def upload(self, field: np.ndarray):
        f = np.ascontiguousarray(field, dtype=np.float64)
        self.N.check(self.L.silt_group_upload(self.h, self.N._dp(f)))

    def begin(self, t_end: float = np.inf, max_steps: int = -1, snapshots=(), dt_cap: int = 0):
        import ctypes as C
        plan, keep = self.N._plan(t_end, max_steps, snapshots, dt_cap)
        self.N.check(self.L.silt_group_begin(self.h, C.byref(plan)))
        del keep

    def step(self, n: int = 1):
        self.N.check(self.L.silt_group_step(self.h, int(n)))

    def status(self):
        import ctypes as C
        st = abi.SiltStatus()
        self.N.check(self.L.silt_group_status(self.h, C.byref(st)))
        return st

    def resume(self):
        self.N.check(self.L.silt_group_resume(self.h))

    def dt_log(self, n: int) -> np.ndarray:
        out = np.empty(n)
        self.N.check(self.L.silt_group_dt_log(self.h, self.N._dp(out), int(n)))
        return out

    def gather(self) -> np.ndarray:
        out = np.empty((self.ny, self.nx, 4))
        self.N.check(self.L.silt_group_download(self.h, self.N._dp(out)))
        return out

    def capture_resume(self, out: np.ndarray):
        """Asynchronous whole-grid snapshot of a paused run (every strip streams
        its rows into ``out`` while the next steps run)."""
        assert out.flags.c_contiguous and out.size == 4 * self.nx * self.ny
        self.N.check(self.L.silt_group_capture_resume(self.h, self.N._dp(out)))

    def capture_wait(self):
        self.N.check(self.L.silt_group_capture_wait(self.h))

    def write_snapshot(self, time: float, path: str) -> int:
        """Whole-grid CSV (write_snapshot), every strip formatted on its device."""
        n = C.c_int64(0)
        self.N.check(self.L.silt_group_write_snapshot(self.h, float(time), os.fsencode(path),
                                                      C.byref(n)))
        return n.value

    def run(self, batch: int = 8, on_snapshot=None, async_snapshots: bool = False):
        return self.N._run_loop(self.step, self.status, self.resume, self.gather,
                                self.capture_resume, self.capture_wait, batch, on_snapshot,
                                async_snapshots, (self.ny, self.nx))

    def close(self):
        if self.h:
            self.L.silt_group_destroy(self.h)
            self.h = None


# ---- two pieces per rank ------------------------------------------------------
# A contiguous strip through the mound is all full-path work: its GPU has no
# quiescent rows for the hot CTAs to overlap with, so on C4 the strips bound
# strong scaling at ~0.77 (N = 8, profiles/r1_strip_balance.md).  Here every
# rank owns TWO row ranges: 1/N of the hot band around the mound and 1/N of the
# far field, stepped as two solvers on two streams of its GPU, so hot and
# quiescent CTAs share the GPU as in the one-GPU launch (tools/strip_times.py
# --pieces: 0.86 at N = 8).  Any layout gives bit-identical fields (the
# reference's layout contract, tests/test_parallel.cpp:215-238).


def piece_partition(row_cost, world: int, spread: int | None = None):
    """Two row ranges per rank: [(hot j0, n), (far j0, n)] for ranks 0..world-1.

    Hot band = the rows of non-quiescent work (row_cost above the quiescent
    level) widened by `spread` rows on both sides (default 2 % of the rows:
    the waves a run sends out), split at equal modelled cost.  The far field
    (the rows below and above the band) is split into `world` pieces of equal
    rows; the pieces BELOW the band go to ranks world//2 .. world-1 and those
    ABOVE to ranks 0 .. world//2 - 1, so no two pieces of one rank are row
    neighbours.  Returns None when the grid has no distinct hot band (then
    contiguous strips are the better layout)."""
    cost = np.asarray(row_cost, dtype=np.float64)
    ny = cost.size
    if world < 2 or ny < 4 * world:
        return None
    quiet = cost.min()
    hot_rows = np.nonzero(cost > quiet * (1 + 1e-9))[0]
    if hot_rows.size == 0:
        return None
    spread = max(1, int(0.02 * ny)) if spread is None else spread
    lo = max(0, int(hot_rows[0]) - spread)
    hi = min(ny, int(hot_rows[-1]) + 1 + spread)
    half = world // 2
    n_lo_pieces, n_hi_pieces = world - half, half
    if hi - lo < world or lo < n_lo_pieces or ny - hi < n_hi_pieces or n_hi_pieces == 0:
        return None
    hot = [(lo + j0, n) for j0, n in balanced_partition(cost[lo:hi], world)]
    out = []
    for r in range(world):
        if r >= half:  # far piece below the band
            j0, n = block_range(lo, n_lo_pieces, r - half)
        else:          # far piece above the band
            j0, n = block_range(ny - hi, n_hi_pieces, r)
            j0 += hi
        out.append([hot[r], (j0, n)])
    return out


def piece_order(layout):
    """All pieces in row order: [(j0, n, rank, k)] (k = 0 hot, 1 far)."""
    pieces = [(j0, n, r, k) for r, ps in enumerate(layout) for k, (j0, n) in enumerate(ps)]
    return sorted(pieces)


class PieceRunner:
    """One rank's pieces (see piece_partition): a CUDA solver per piece on its
    own stream, exchanging over peer memory with every piece of every rank
    ("virtual ranks" = pieces in row order).  Per step, with no host
    synchronisation: each piece's step kernel stores its edge rows into the
    neighbouring pieces' receive rows and its axis-speed maxima into every
    piece's slot, and waits (bounded) for every piece's previous step before
    it starts — exactly the StripRunner peer-memory protocol, with 2N
    participants.  Requires peer memory (CUDA IPC); 2D, non-periodic y."""

    def __init__(self, problem, world: int, rank: int, layout, device: int = 0,
                 variant: int = abi.VARIANT_FAST):
        import torch
        import torch.distributed as dist
        from . import native
        if problem.dim != 2 or problem.bc[abi.SOUTH].type == abi.BC_PERIODIC:
            raise ValueError("pieces: 2D grids with non-periodic y only")
        self.problem, self.world, self.rank = problem, world, rank
        self.layout = layout
        self._dist = dist
        self.device = torch.device("cuda", device)
        order = piece_order(layout)
        self.vworld = len(order)
        vid = {(r, k): v for v, (_, _, r, k) in enumerate(order)}
        self.pieces = []
        # the hot piece runs 32-row blocks (tools/strip_times.py --pieces: 32
        # beat the launch-size default, 8 and 16 on C4 at N = 4 and 8);
        # SILT_ROWS set by the caller wins
        hot_rows = os.environ.get("SILT_PIECE_HOT_ROWS", "32")
        for k, (j0, n) in enumerate(layout[rank]):
            v = vid[(rank, k)]
            south = v - 1 if v > 0 else None
            north = v + 1 if v < self.vworld - 1 else None
            strip = abi.SiltStrip(j0, n, int(south is not None), int(north is not None))
            user_rows = os.environ.get("SILT_ROWS")
            if k == 0 and user_rows is None and hot_rows != "0":
                os.environ["SILT_ROWS"] = hot_rows
            try:
                s = native.Solver(problem, strip, device, variant)
            finally:
                if user_rows is None:
                    os.environ.pop("SILT_ROWS", None)
            st = torch.cuda.Stream(device=device)
            s.set_stream(st.cuda_stream)
            self.pieces.append({"j0": j0, "n": n, "v": v, "south": south, "north": north,
                                "solver": s, "stream": st})
        # handshake: every piece's handles, in virtual-rank order
        mine = [(p["v"], p["solver"].p2p_export()) for p in self.pieces]
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        handles = [None] * self.vworld
        for lst in allh:
            for v, h in lst:
                handles[v] = h
        ok = 1
        try:
            for p in self.pieces:
                p["solver"].p2p_connect(p["v"], self.vworld, handles, p["south"], p["north"])
        except Exception:
            ok = 0
        t = torch.tensor([ok], dtype=torch.int32, device=self._reduce_device())
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) != 1:
            for p in self.pieces:
                p["solver"].close()
            self.pieces = []
            raise RuntimeError("pieces: peer-memory connection failed on some rank")
        self.torch_stream = torch.cuda.Stream(device=device)  # joins the pieces' streams
        self.j0 = min(p["j0"] for p in self.pieces)
        self.nrows = sum(p["n"] for p in self.pieces)
        self._p2p = True

    def _reduce_device(self):
        return "cpu" if self._dist.get_backend() == "gloo" else self.device

    # ---- run control ------------------------------------------------------
    def upload_rows(self, rows_fn):
        """rows_fn(j0, n) -> device tensor (n, nx, 4) of the piece's initial rows."""
        import torch
        for p in self.pieces:
            t = rows_fn(p["j0"], p["n"])
            torch.cuda.current_stream(self.device).synchronize()
            p["solver"].upload_device(t.data_ptr())
            p["stream"].synchronize()

    def upload_host(self, full):
        """Rows of the WHOLE grid (host array); each piece takes its own."""
        for p in self.pieces:
            p["solver"].upload(np.ascontiguousarray(full[p["j0"]:p["j0"] + p["n"]]))

    def upload_host_tensors(self, tensors):
        """One (n, nx, 4) host tensor per piece (pinned: the copy is async)."""
        from .native import check
        for p, t in zip(self.pieces, tensors):
            s = p["solver"]
            check(s.L.silt_solver_upload(s.h, C.cast(t.data_ptr(), C.POINTER(C.c_double))))

    def download_host_tensors(self, tensors):
        from .native import check
        for p, t in zip(self.pieces, tensors):
            s = p["solver"]
            check(s.L.silt_solver_download(s.h, C.cast(t.data_ptr(), C.POINTER(C.c_double))))

    def begin(self, t_end: float = np.inf, max_steps: int = -1, snapshots=(), dt_cap: int = 0):
        import torch
        if snapshots:
            raise ValueError("pieces: snapshots are not supported (use StripRunner)")
        for p in self.pieces:
            p["solver"].begin(t_end=t_end, max_steps=max_steps, dt_cap=dt_cap)
        # global MAX of the initial axis speeds over every piece (global_dt,
        # src/parallel.cpp:200-206); the initial reduction kernels delivered
        # the edge rows themselves
        slots = [torch.as_tensor(_CAI(p["solver"].reduce_slot(), 2), device=self.device)
                 for p in self.pieces]
        for p in self.pieces:
            p["stream"].synchronize()
        m = torch.stack(slots).max(dim=0).values
        dev = self._reduce_device()
        m = m.to(dev)
        self._dist.all_reduce(m, op=self._dist.ReduceOp.MAX)
        m = m.to(self.device)
        for s in slots:
            s.copy_(m)
        torch.cuda.synchronize(self.device)

    def step(self, n: int = 1):
        for _ in range(n):
            for p in self.pieces:
                p["solver"].p2p_step(1)

    def record_join(self):
        """Make torch_stream wait for every piece's stream (for events)."""
        for p in self.pieces:
            self.torch_stream.wait_stream(p["stream"])

    def synchronize(self):
        for p in self.pieces:
            p["stream"].synchronize()

    def status(self):
        sts = [p["solver"].status() for p in self.pieces]
        return sts[0]

    def launch_count(self) -> int:
        return sum(p["solver"].launch_count() for p in self.pieces)

    def barrier(self):
        self._dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64, device=self._reduce_device())
        self._dist.all_reduce(t, op=self._dist.ReduceOp.MAX)
        return float(t.item())

    def dt_log(self, n: int):
        return self.pieces[0]["solver"].dt_log(n)

    def gather(self):
        """The global field on rank 0 (every piece's rows at its offset)."""
        mine = [(p["j0"], p["solver"].download()) for p in self.pieces]
        parts = [None] * self.world if self.rank == 0 else None
        self._dist.gather_object(mine, parts, dst=0)
        if self.rank != 0:
            return None
        ny, nx = self.problem.ny, self.problem.nx
        out = np.empty((ny, nx, 4))
        for lst in parts:
            for j0, a in lst:
                out[j0:j0 + a.shape[0]] = a
        return out

    def close(self):
        # peers may still be storing into this rank's memory: drain, then
        # every rank frees together
        self.synchronize()
        self._dist.barrier()
        for p in self.pieces:
            p["solver"].close()
        self.pieces = []

    def shutdown(self):
        if self._dist.is_initialized():
            self._dist.destroy_process_group()
