"""Row-partitioned pipelined CG (BASELINE configs[3]).

The global system is ``gen_poisson3d_block(side, 1)`` (reference io.py:232-275;
values 12/-2, b = ones unless given, x0 = 0), solved with the reference's
pipelined CG recurrences (solvers.py:395-469) at the one-element-per-lane
geometry ``ExecutionContext(n_groups, group_size)`` with
``n_groups * group_size == n``.  The rows are split into ``world``
group-aligned z-slabs; per iteration the library exchanges one z-plane of the
recompute-at-gather inputs (r, p, Ap) with each neighbour, runs the fused CG
kernel on the local rows, allgathers the group partials once and runs the same
serial stage 2 on every rank.  Results are bit-identical to
``cg_pipelined(gen_poisson3d_block(side, 1), b, context=...)`` on one device.

Two transports (pipekrylov_b200.h, pk_dcg_*):

* ``cg_partitioned(side, world, ...)`` -- all partitions in this process on one
  device (halo = device copies); the bit-exactness proof on a single GPU;
* ``PartitionedCG(side, group_size, rank=, world=)`` under ``torchrun`` -- one
  partition per process and GPU, NCCL send/recv halos and an in-place NCCL
  allgather (the communicator is created by the library from a unique id
  that rank 0 broadcasts with ``torch.distributed``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .device import context_for
from .linalg import ExecutionContext
from .solvers import SolverConfig, SolverResult, _native_config, _trace_from


def slab_geometry(side: int, group_size: int) -> ExecutionContext:
    """The one-element-per-lane geometry for a side^3 grid."""
    n = side ** 3
    if n % group_size:
        raise ValueError("group_size must divide side^3")
    return ExecutionContext(n_groups=n // group_size, group_size=group_size)


def _result(res, x, hist, n):
    return SolverResult(
        x=x, residual_history=[float(v) for v in hist[: res.iterations]],
        true_final_residual=float(res.true_final_residual), iterations=int(res.iterations),
        termination=N.TERM_NAMES[res.termination], trace=_trace_from(res, "cg", n, 30),
        breakdown_kind=N.KIND_NAMES[res.breakdown_kind], loop_seconds=float(res.loop_seconds),
        diagnostics={"launches_per_iteration": int(res.launches_per_iteration)})


class _Handle:
    def __init__(self, dc, side, geom, world, rank, comm, limit):
        h = C.c_void_p()
        N.check(N.lib().pk_dcg_create(dc.handle, side, geom.n_groups, geom.group_size, world, rank, comm,
                                      max(limit, 1), C.byref(h)), "pk_dcg_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            N.lib().pk_dcg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cg_partitioned(side: int, world: int, group_size: int, b=None, config=None, device: int = 0) -> SolverResult:
    """All `world` partitions in this process on one device."""
    cfg = SolverConfig.coerce(config)
    geom = slab_geometry(side, group_size)
    n = side ** 3
    limit = cfg.iteration_limit()
    dc = context_for(ExecutionContext(geom.n_groups, geom.group_size, device=device))
    dc.reset_stream()
    h = _Handle(dc, side, geom, world, 0, None, limit)
    try:
        bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        if bb is not None and bb.shape != (n,):
            raise ValueError(f"b has shape {bb.shape}, expected ({n},)")
        x = np.empty(n)
        hist = np.empty(max(limit, 1))
        res = N.PkResult()
        dp = C.POINTER(C.c_double)
        N.check(N.lib().pk_dcg_solve(h.h, bb.ctypes.data_as(dp) if bb is not None else None,
                                     C.byref(_native_config(cfg)), x.ctypes.data_as(dp), hist.ctypes.data_as(dp),
                                     len(hist), C.byref(res)), "pk_dcg_solve")
        return _result(res, x, hist, n)
    finally:
        h.close()


class PartitionedCG:
    """One partition per process (torchrun): NCCL halos and allgather.

    ``torch.distributed`` must be initialised; rank 0's NCCL unique id is
    broadcast through it.  ``solve()`` returns the SolverResult with this
    rank's rows of x (rows [rank n/world, (rank+1) n/world))."""

    def __init__(self, side: int, group_size: int, rank: int, world: int, device: int, limit: int):
        import torch
        import torch.distributed as dist

        self.side, self.rank, self.world, self.device = side, rank, world, device
        self.geom = slab_geometry(side, group_size)
        self.n = side ** 3
        self.nloc = self.n // world
        self.limit = limit
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            N.check(N.lib().pk_nccl_unique_id(C.cast(uid, C.c_void_p)), "pk_nccl_unique_id")
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=f"cuda:{device}")
        dist.broadcast(t, src=0)
        raw = bytes(t.cpu().tolist())
        uid2 = (C.c_ubyte * 128).from_buffer_copy(raw)
        comm = C.c_void_p()
        N.check(N.lib().pk_nccl_comm_create(device, C.cast(uid2, C.c_void_p), world, rank, C.byref(comm)),
                "pk_nccl_comm_create")
        self.comm = comm
        self.dc = context_for(ExecutionContext(self.geom.n_groups, self.geom.group_size, device=device))
        self.dc.reset_stream()
        self.h = _Handle(self.dc, side, self.geom, world, rank, comm, limit)

    def solve(self, config=None, b_local=None) -> SolverResult:
        cfg = SolverConfig.coerce(config)
        if cfg.iteration_limit() > self.limit:
            raise ValueError("iteration limit exceeds the capacity given at construction")
        x = np.empty(self.nloc)
        hist = np.empty(max(self.limit, 1))
        res = N.PkResult()
        dp = C.POINTER(C.c_double)
        bb = None if b_local is None else np.ascontiguousarray(b_local, dtype=np.float64)
        if bb is not None and bb.shape != (self.nloc,):
            raise ValueError(f"b_local must have shape ({self.nloc},), got {bb.shape}")
        N.check(N.lib().pk_dcg_solve(self.h.h, bb.ctypes.data_as(dp) if bb is not None else None,
                                     C.byref(_native_config(cfg)), x.ctypes.data_as(dp), hist.ctypes.data_as(dp),
                                     len(hist), C.byref(res)), "pk_dcg_solve")
        return _result(res, x, hist, self.n)

    def close(self):
        self.h.close()
        if self.comm:
            N.lib().pk_nccl_comm_destroy(self.comm)
            self.comm = None
