"""Parity at the BASELINE config sizes against the REAL reference.

Fixtures: tests/golden/scale_manifest.json + tests/golden/scale/*.npz,
written by tests/golden/make_scale_golden.py, which ran the reference's own
pipelined drivers (pipekrylov.SOLVERS) on these systems in the development
container.  Each case stores the residual history, iterations, termination,
true residual and the SHA-256 of the whole solution vector, so the checks
below are bit-for-bit over every entry of x without committing megabytes:

* C4 (CG 3D Poisson): 128^3 to tolerance at the slab geometry 512 x 4096,
  through the row-partitioned solver with 1/2/4/8 partitions (halo + one
  partials allgather per iteration), and 256^3 over 30 fixed iterations at
  256 x 65536 (1/2/4/8 partitions);
* C4 at the reference's DEFAULT geometry 128 x 256: bitwise on one device,
  and the north-star bar for the partitioned solver (which must use the
  one-element-per-lane slab geometry): +-1 iteration, 1e-10 relative history
  and solution;
* C3 (GMRES(30) 3D conv-diff 128^3): 31 fixed steps (a whole cycle: ξ stage
  2, host triangular solve, x update, restart) and to tolerance (true-residual
  gate) at 64^3 / 128^3 when the fixture exists;
* C2 (BiCGStab 2D conv-diff 1024^2) to tolerance (2389 iterations);
* BiCGStab runs whose residual identity clamps below tol, so the
  reference's "check" phase runs -- passing, and failing then resuming;
* the NCCL transport of the partitioned solver with one rank.
"""

from __future__ import annotations

import hashlib
import json
import os
import socket
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def pk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1410_4054_b200 as pk

    return pk


@lru_cache(maxsize=None)
def manifest():
    return json.loads((GOLD / "scale_manifest.json").read_text())["cases"]


def case(name):
    if name not in manifest():
        pytest.skip(f"fixture {name} not generated")
    return manifest()[name], dict(np.load(GOLD / "scale" / f"{name}.npz"))


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def assert_bitwise(res, name):
    meta, store = case(name)
    assert res.iterations == meta["iterations"], (res.iterations, meta["iterations"])
    assert res.termination == meta["termination"]
    assert res.breakdown_kind == meta["breakdown_kind"]
    assert np.array_equal(bits(res.residual_history), bits(store["history"]))
    assert sha(res.x) == meta["x_sha256"]
    assert res.true_final_residual == float(store["true_final_residual"][0])


def history_gap(h1, h2, floor=1e-12):
    """Max relative gap of two histories, entries below the reference's
    1e-12 noise floor ignored (test_acceptance.py:43, 66-73)."""
    worst = 0.0
    for x, y in zip(h1, h2):
        if abs(x) <= floor and abs(y) <= floor:
            continue
        worst = max(worst, abs(x - y) / max(abs(x), abs(y)))
    return worst


# ---------------------------------------------------------------------------
# C4: CG 3D Poisson, row-partitioned
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_c4_128_to_tolerance_partitioned_bitwise(pk, world):
    res = pk.cg_partitioned(128, world, 4096, config=pk.SolverConfig(max_iterations=2000))
    assert_bitwise(res, "c4_128_tol_slab")


def test_c4_128_default_geometry_single_device_bitwise(pk):
    dm, b = pk.poisson3d_grid(128, device=True)
    res = pk.cg_pipelined(dm, b, config=pk.SolverConfig(max_iterations=2000), context=pk.ExecutionContext(128, 256))
    assert_bitwise(res, "c4_128_tol_default")


def test_c4_128_partitioned_vs_default_geometry_reference(pk):
    """The partitioned solver needs the one-element-per-lane slab geometry;
    against the reference run at its DEFAULT geometry the north-star bar
    holds: +-1 iteration, history and x within 1e-10 relative."""
    meta, store = case("c4_128_tol_default")
    res = pk.cg_partitioned(128, 4, 4096, config=pk.SolverConfig(max_iterations=2000))
    assert abs(res.iterations - meta["iterations"]) <= 1
    gap = history_gap(res.residual_history, store["history"])
    xs = np.asarray(res.x)[store["x_idx"]]
    xerr = np.abs(xs - store["x_sample"]).max() / np.abs(store["x_sample"]).max()
    print(f"c4 128^3 slab vs default geometry: dit={res.iterations - meta['iterations']} "
          f"history gap={gap:.3e} x rel err (sample)={xerr:.3e}")
    assert gap <= 1e-10
    assert xerr <= 1e-10


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_c4_256_fixed30_partitioned_bitwise(pk, world):
    cfg = pk.SolverConfig(fixed_iterations=30, max_iterations=30)
    res = pk.cg_partitioned(256, world, 65536, config=cfg)
    assert_bitwise(res, "c4_256_fixed30_slab")


# ---------------------------------------------------------------------------
# C3: GMRES(30) 3D convection-diffusion
# ---------------------------------------------------------------------------


def test_c3_128_full_cycle_and_restart_bitwise(pk):
    dm, b = pk.convdiff3d(128, device=True)
    cfg = pk.SolverConfig(fixed_iterations=31, max_iterations=31, restart=30)
    res = pk.gmres_pipelined(dm, b, config=cfg)
    assert_bitwise(res, "c3_128_fixed31")


@pytest.mark.parametrize("side", [64, 128])
def test_c3_to_tolerance_bitwise(pk, side):
    meta, _ = case(f"c3_{side}_tol")
    dm, b = pk.convdiff3d(side, device=True)
    res = pk.gmres_pipelined(dm, b, config=pk.SolverConfig(**meta["config"]))
    assert_bitwise(res, f"c3_{side}_tol")


# ---------------------------------------------------------------------------
# C2: BiCGStab 2D convection-diffusion; the check phase
# ---------------------------------------------------------------------------


def test_c2_1024_to_tolerance_bitwise(pk):
    dm, b = pk.convdiff2d(1024, device=True)
    res = pk.bicgstab_pipelined(dm, b, config=pk.SolverConfig(max_iterations=20000))
    assert_bitwise(res, "c2_1024_tol")


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("name", ["bicgstab_check_pass", "bicgstab_check_resume", "bicgstab_check_resume_g1x4"])
def test_bicgstab_check_phase_bitwise(pk, name, split, monkeypatch):
    """The clamped-identity "check" phase (solvers.py:687-694), passing and
    failing-then-resuming; split = 1 forces the split body, which on these
    CHAIN geometries runs as the persistent cooperative loop -- relaunched
    after every failed check."""
    monkeypatch.setenv("PK_BICG_SPLIT", split)
    meta, store = case(name)
    spec = json.loads((GOLD / "scale_check_spec.json").read_text())[name]
    a = pk.CsrMatrix.from_dense(spec["dense"])
    res = pk.bicgstab_pipelined(a, np.asarray(spec["b"]), config=pk.SolverConfig(**spec["config"]),
                                context=pk.ExecutionContext(*spec["geom"]))
    assert_bitwise(res, name)
    assert np.array_equal(bits(res.x), bits(store["x"]))
    assert [p.label for p in res.trace.phases].count("check") == meta["check_phases"] >= 1


# ---------------------------------------------------------------------------
# NCCL transport, one rank
# ---------------------------------------------------------------------------


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partitioned_cg_nccl_transport_world1(pk):
    """PartitionedCG over a real NCCL communicator (halo send/recv with no
    neighbour, in-place allgather of the partials) equals the in-process
    partitioned solver bit for bit."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        side, gs = 32, 1024
        cfg = pk.SolverConfig(max_iterations=400)
        solver = pk.PartitionedCG(side, gs, 0, 1, 0, 400)
        try:
            res = solver.solve(cfg)
        finally:
            solver.close()
    finally:
        dist.destroy_process_group()
    ref = pk.cg_partitioned(side, 1, gs, config=cfg)
    assert res.iterations == ref.iterations and res.termination == ref.termination
    assert np.array_equal(bits(res.residual_history), bits(ref.residual_history))
    assert np.array_equal(bits(res.x), bits(ref.x))
    assert res.true_final_residual == ref.true_final_residual
