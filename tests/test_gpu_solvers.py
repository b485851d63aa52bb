"""Solver-level parity on the B200 through the reference-facing API.

* every golden case produced by the real reference (tests/golden): iterations,
  termination, breakdown kind, residual history, x and the true residual must
  be bit-identical;
* larger systems and other geometries against the oracle, bitwise;
* the BASELINE configs at full size: C1 (CG 512^2, to tolerance) and C2
  (BiCGStab 1024^2) / C3 (GMRES(30) 128^3) over fixed iterations, bitwise
  against the oracle, plus the north-star tolerance bar (+-1 iteration,
  1e-10 relative) against the oracle at the reference's default geometry;
* graph vs host loop, reruns, device generators."""

import numpy as np
import pytest

from oracle import pk_oracle as orc
from tests import golden_data as gd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1410_4054_b200 as pk

    return pk


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(bits(a), bits(b))


def assert_identical(res, ref):
    assert res.iterations == ref["iterations"]
    assert res.termination == ref["termination"]
    assert res.breakdown_kind == ref["breakdown_kind"]
    assert same(res.residual_history, ref["history"])
    assert same(res.x, ref["x"])
    assert res.true_final_residual == ref["true_final_residual"]


@pytest.mark.parametrize("name", gd.solver_case_names())
def test_solver_matches_reference_golden(pk, name):
    case = gd.solver_case(name)
    store = gd.solvers()
    a = pk.CsrMatrix(*gd.csr_arrays(store, f"{name}/A"))
    b = store[f"{name}/b"]
    x0 = store.get(f"{name}/x0")
    cfg = pk.SolverConfig(**case["config"])
    ctx = pk.ExecutionContext(*case["geom"])
    res = pk.SOLVERS[(case["method"], "pipelined")](a, b, x0=x0, config=cfg, context=ctx)
    ref = {"iterations": case["iterations"], "termination": case["termination"],
           "breakdown_kind": case["breakdown_kind"], "history": store[f"{name}/history"],
           "x": store[f"{name}/x"], "true_final_residual": store[f"{name}/true_final_residual"][0]}
    assert_identical(res, ref)


def oracle_run(method, a, b, geom, **kw):
    return orc.SOLVERS[method](a, b, geom=geom, **kw)


@pytest.mark.parametrize("name", gd.classical_case_names())
def test_classical_matches_reference_golden(pk, name):
    """SOLVERS[(m, "classical")] on the B200 kernels (pk_spmv / pk_dot /
    pk_vec_update) vs the reference's classical drivers, bitwise."""
    case = gd.classical_case(name)
    store = gd.classical()
    a = pk.CsrMatrix(*gd.csr_arrays(store, f"{name}/A"))
    b = store[f"{name}/b"]
    x0 = store.get(f"{name}/x0")
    cfg = pk.SolverConfig(**case["config"])
    ctx = pk.ExecutionContext(*case["geom"])
    res = pk.SOLVERS[(case["method"], "classical")](a, b, x0=x0, config=cfg, context=ctx)
    ref = {"iterations": case["iterations"], "termination": case["termination"],
           "breakdown_kind": case["breakdown_kind"], "history": store[f"{name}/history"],
           "x": store[f"{name}/x"], "true_final_residual": store[f"{name}/true_final_residual"][0]}
    assert_identical(res, ref)


@pytest.mark.parametrize("method", ["cg", "bicgstab", "gmres"])
def test_classical_matches_oracle_medium(pk, method):
    """Classical drivers on a 120^2 system vs the oracle's classical
    restatement at two geometries (incl. MGS for GMRES)."""
    a, _ = pk.convdiff2d(120) if method != "cg" else pk.poisson2d_grid(120)
    b = np.random.default_rng(2).random(a.n_rows)
    for geom in ((128, 256), (16, 1024)):
        for mgs in ((False, True) if method == "gmres" else (False,)):
            kw = {"orthogonalization": "modified_gs"} if mgs else {}
            res = pk.SOLVERS[(method, "classical")](a, b, config=pk.SolverConfig(max_iterations=200, **kw),
                                                     context=pk.ExecutionContext(*geom))
            okw = {"mgs": mgs} if method == "gmres" else {}
            assert_identical(res, orc.CLASSICAL[method](a, b, geom=geom, max_iterations=200, **okw))


@pytest.mark.parametrize("method", ["cg", "bicgstab", "gmres"])
@pytest.mark.parametrize("geom", [(128, 256), (32, 1024), (1, 4096), (16, 65536), (1000, 64)])
def test_solver_matches_oracle_medium(pk, method, geom):
    a, _ = pk.convdiff2d(120) if method != "cg" else pk.poisson2d_grid(120)
    b = np.random.default_rng(1).random(a.n_rows)
    res = pk.SOLVERS[(method, "pipelined")](a, b, config=pk.SolverConfig(max_iterations=300),
                                             context=pk.ExecutionContext(*geom))
    assert_identical(res, oracle_run(method, a, b, geom, max_iterations=300))


@pytest.mark.parametrize("mode", ["graph", "host"])
def test_loop_modes_identical(pk, mode):
    a, b = pk.poisson2d_grid(64)
    cfg = pk.SolverConfig(loop_mode=mode)
    for method in ("cg", "bicgstab"):
        res = pk.SOLVERS[(method, "pipelined")](a, b, config=cfg)
        assert_identical(res, oracle_run(method, a, b, (128, 256)))


@pytest.mark.parametrize("unroll", ["1", "3", "8"])
def test_graph_unroll_identical(pk, unroll, monkeypatch):
    """Iterations per WHILE-body execution (PK_UNROLL, read when the loop
    graph is built): stops inside an unrolled body must leave no trace --
    converged, max_iter and fixed-iteration runs with iteration counts that
    are not multiples of the unroll."""
    monkeypatch.setenv("PK_UNROLL", unroll)
    a, b = pk.poisson2d_grid(50)
    for method, kw, okw in (("cg", {}, {}), ("bicgstab", {}, {}), ("cg", {"max_iterations": 13}, {"max_iterations": 13}),
                            ("bicgstab", {"fixed_iterations": 7, "max_iterations": 7}, {"fixed": 7, "max_iterations": 7})):
        res = pk.SOLVERS[(method, "pipelined")](a, b, config=pk.SolverConfig(**kw))
        assert_identical(res, oracle_run(method, a, b, (128, 256), **okw))


@pytest.mark.parametrize("split", ["0", "1"])
def test_split_and_fused_bodies_identical(pk, split, monkeypatch):
    """Loop bodies: fused recompute-at-gather kernels (OpCgFused / OpBicgA)
    or the update sweep + one-gather SpMV (default for n >= 2^20) -- forced
    both ways here on a medium system; bits and iteration counts unchanged,
    launches per iteration 1/2 (CG) and 2/3 (BiCGStab)."""
    monkeypatch.setenv("PK_CG_SPLIT", split)
    monkeypatch.setenv("PK_BICG_SPLIT", split)
    a, b = pk.convdiff2d(96)
    pa, pb = pk.poisson2d_grid(96)
    for method, A, B in (("cg", pa, pb), ("bicgstab", a, b)):
        for kw, okw in (({}, {}), ({"fixed_iterations": 9, "max_iterations": 9}, {"fixed": 9, "max_iterations": 9})):
            res = pk.SOLVERS[(method, "pipelined")](A, B, config=pk.SolverConfig(**kw))
            assert_identical(res, oracle_run(method, A, B, (128, 256), **okw))
            want = {"cg": 1, "bicgstab": 2}[method] + (split == "1")
            assert [p.launches for p in res.trace.iterations[:3]] == [want] * 3


@pytest.mark.parametrize("geom", [(8, 64), (4, 32), (2, 512)])
def test_two_phase_engine_identical(pk, geom, monkeypatch):
    """Two-phase SpMV engine (opt-in, PK_MAT_MINK read at context creation;
    compiled in with -DPK_MAT_ENGINE, otherwise the default engines run under
    the same setting): thread-per-row pass storing the contributions, then the
    ordered lane-chain fold.  Geometries cover a group spanning several fold
    CTAs (2 x 512), one (8 x 64) and several groups per fold CTA (4 x 32);
    chains K >= 9.  Bits, iteration counts and termination identical to the
    oracle."""
    monkeypatch.setenv("PK_MAT_MINK", "9")
    a, b = pk.convdiff2d(96)
    pa, pb = pk.poisson2d_grid(96)
    ctx = pk.ExecutionContext(*geom, device=0)
    for method, A, B in (("cg", pa, pb), ("bicgstab", a, b), ("gmres", a, b)):
        for kw, okw in (({}, {}), ({"fixed_iterations": 9, "max_iterations": 9}, {"fixed": 9, "max_iterations": 9})):
            res = pk.SOLVERS[(method, "pipelined")](A, B, config=pk.SolverConfig(**kw), context=ctx)
            assert_identical(res, oracle_run(method, A, B, geom, **okw))


def test_reruns_bit_identical(pk):
    a, b = pk.convdiff2d(80)
    for key, solver in pk.SOLVERS.items():
        r1, r2 = solver(a, b), solver(a, b)
        assert r1.residual_history == r2.residual_history and same(r1.x, r2.x)
        assert [(p.label, p.launches) for p in r1.trace.phases] == [(p.label, p.launches) for p in r2.trace.phases]


def test_trace_shape_and_counts(pk):
    a, b = pk.gen_poisson2d(1)
    cfg = pk.SolverConfig(fixed_iterations=5, max_iterations=5)
    cg = pk.cg_pipelined(a, b, config=cfg)
    # reference (emulated): CG 2 launches + 1 transfer, BiCGStab 4 + 1
    # (test_acceptance.py:85-108).  B200: the update is folded into the SpMV
    # (recompute-at-gather) and stage 2 runs on the device.
    assert [p.launches for p in cg.trace.iterations] == [1] * 5
    assert all(p.transfers == 0 for p in cg.trace.iterations)  # device-resident loop
    bi = pk.bicgstab_pipelined(a, b, config=cfg)
    # small system: fused bodies (n >= 2^20 splits the update off: CG 2,
    # BiCGStab 3 -- test_split_and_fused_bodies_identical)
    assert [p.launches for p in bi.trace.iterations] == [2] * 5
    gm = pk.gmres_pipelined(a, b, config=cfg)
    assert [p.launches for p in gm.trace.iterations] == [2, 3, 4, 4, 4]
    for r in (cg, bi, gm):
        labels = [p.label for p in r.trace.phases]
        assert labels[0] == "setup" and labels[-1] == "finish"


def test_solve_entry_point(pk):
    a, b = pk.gen_poisson2d(2)
    res = pk.solve(a, b, tag="cg", tol=1e-8, maxiter=500)
    assert res.converged and res.true_final_residual <= 1e-8 * np.linalg.norm(b)
    res2 = pk.solve(a, b, tag=("gmres", "pipelined"), tol=1e-8, maxiter=500)
    assert res2.converged


def test_reference_objects_accepted(pk):
    # duck-typed reference CsrMatrix / SolverConfig / ExecutionContext
    class RefCsr:
        def __init__(self, m):
            self.n_rows, self.n_cols = m.n_rows, m.n_cols
            self.row_offsets, self.col_indices, self.values = m.rowptr, m.cols, m.vals

    class RefCtx:
        n_groups, group_size = 16, 32

    o, b = orc.poisson2d(2)
    res = pk.cg_pipelined(RefCsr(o), b, context=RefCtx())
    assert_identical(res, oracle_run("cg", o, b, (16, 32)))


@pytest.mark.parametrize("fam,dims", [("poisson2d", (37,)), ("poisson3d", (11,)), ("convdiff2d", (45,)),
                                      ("convdiff3d", (13,))])
def test_device_generators_equal_host(pk, fam, dims):
    host_fn = {"poisson2d": pk.poisson2d_grid, "poisson3d": pk.poisson3d_grid, "convdiff2d": pk.convdiff2d,
               "convdiff3d": pk.convdiff3d}[fam]
    ha, _ = host_fn(*dims)
    dm, _ = host_fn(*dims, device=True)
    back = dm.download(pk.context_for(pk.ExecutionContext()))
    assert np.array_equal(back.row_offsets, ha.row_offsets) and np.array_equal(back.col_indices, ha.col_indices)
    assert same(back.values, ha.values)
    assert dm.max_row_nnz == int(ha.row_nnz().max())


def test_device_matrix_solve_equals_host_matrix_solve(pk):
    dm, b = pk.convdiff2d(90, device=True)
    ha, _ = pk.convdiff2d(90)
    r1 = pk.bicgstab_pipelined(dm, b)
    r2 = pk.bicgstab_pipelined(ha, b)
    assert r1.residual_history == r2.residual_history and same(r1.x, r2.x)


# ---------------------------------------------------------------------------
# BASELINE configurations at full size
# ---------------------------------------------------------------------------


def history_gap(h1, h2, floor=1e-12):
    worst = 0.0
    for x, y in zip(h1, h2):
        if abs(x) <= floor and abs(y) <= floor:
            continue
        worst = max(worst, abs(x - y) / max(abs(x), abs(y)))
    return worst


def test_c1_cg_512_to_tolerance_bitwise(pk):
    """C1: pipelined CG, 2D Poisson 512x512, tol 1e-8 (oracle: 941 iterations)."""
    a, b = pk.poisson2d_grid(512)
    res = pk.cg_pipelined(a, b, config=pk.SolverConfig(max_iterations=2000))
    ref = oracle_run("cg", a, b, (128, 256), max_iterations=2000)
    assert ref["iterations"] == 941
    assert_identical(res, ref)
    # north-star bar, stated explicitly: +-1 iteration, 1e-10 relative
    assert abs(res.iterations - ref["iterations"]) <= 1
    assert history_gap(res.residual_history, ref["history"]) <= 1e-10
    assert np.abs(res.x - ref["x"]).max() / np.abs(ref["x"]).max() <= 1e-10


def test_c1_wide_geometry_matches_oracle_same_geometry(pk):
    a, b = pk.poisson2d_grid(512)
    ctx = pk.ExecutionContext.one_per_lane(a.n_rows, 1024)
    res = pk.cg_pipelined(a, b, config=pk.SolverConfig(max_iterations=2000), context=ctx)
    assert_identical(res, oracle_run("cg", a, b, (ctx.n_groups, ctx.group_size), max_iterations=2000))


def test_c2_bicgstab_1024_fixed_bitwise(pk):
    """C2 shape: BiCGStab 2D upwind convection-diffusion 1024^2, 8 fixed iterations."""
    dm, b = pk.convdiff2d(1024, device=True)
    a, _ = pk.convdiff2d(1024)
    cfg = pk.SolverConfig(fixed_iterations=8, max_iterations=8)
    res = pk.bicgstab_pipelined(dm, b, config=cfg)
    assert_identical(res, oracle_run("bicgstab", a, b, (128, 256), fixed=8, max_iterations=8))
    assert [p.launches for p in res.trace.iterations[:2]] == [0, 0]  # split body at n = 2^20: one persistent kernel


def test_c3_gmres_128_fixed_bitwise(pk):
    """C3 shape: GMRES(30) 3D upwind convection-diffusion 128^3, 6 fixed steps."""
    dm, b = pk.convdiff3d(128, device=True)
    a, _ = pk.convdiff3d(128)
    cfg = pk.SolverConfig(fixed_iterations=6, max_iterations=6)
    res = pk.gmres_pipelined(dm, b, config=cfg)
    assert_identical(res, oracle_run("gmres", a, b, (128, 256), fixed=6, max_iterations=6))


# ---------------------------------------------------------------------------
# C5: transient batch of independent systems
# ---------------------------------------------------------------------------


def test_c5_batch_each_system_bitwise(pk):
    """configs[4] in miniature: mixed sizes, distinct seeded RHS; every system
    of the batch equals its own single solve and the oracle, bitwise."""
    sides = [15, 31, 63, 31, 15, 47, 63, 15]
    mats = {s: pk.poisson2d_grid(s)[0] for s in set(sides)}
    systems = [(mats[s], np.random.default_rng(i).random(s * s)) for i, s in enumerate(sides)]
    ctx = pk.ExecutionContext(4, 64)
    out = pk.solve_batch(systems, tag="cg", config=pk.SolverConfig(max_iterations=400), context=ctx, threads=3)
    assert len(out) == len(systems)
    for i, ((a, b), r) in enumerate(zip(systems, out)):
        single = pk.cg_pipelined(a, b, config=pk.SolverConfig(max_iterations=400), context=ctx)
        assert r.iterations == single.iterations and same(r.x, single.x)
        assert same(r.residual_history, single.residual_history)
        if i < 3:
            assert_identical(r, oracle_run("cg", a, b, (4, 64), max_iterations=400))


@pytest.mark.parametrize("tag", ["bicgstab", "gmres"])
def test_batch_other_drivers(pk, tag):
    a, b = pk.convdiff2d(24)
    systems = [(a, b * (1.0 + k)) for k in range(4)]
    out = pk.solve_batch(systems, tag=tag, config=pk.SolverConfig(max_iterations=300), threads=2)
    for (aa, bb), r in zip(systems, out):
        single = pk.SOLVERS[(tag, "pipelined")](aa, bb, config=pk.SolverConfig(max_iterations=300))
        assert r.iterations == single.iterations and same(r.x, single.x)


# ---------------------------------------------------------------------------
# C4: row-partitioned CG (in-process partitions on one device)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_c4_partitioned_cg_bitwise(pk, world, split, monkeypatch):
    """gen_poisson3d_block(32, 1) split into `world` z-slabs: halo exchange +
    one partials allgather per iteration reproduce the single-device oracle at
    the same geometry bit for bit; both loop forms (fused
    step with r/p/Ap halos, or update sweep + p' halo + SpMV -- the default
    for partitions >= 2^20 rows)."""
    monkeypatch.setenv("PK_CG_SPLIT", split)
    side, gs = 32, 1024
    geom = pk.slab_geometry(side, gs)
    a, b = pk.gen_poisson3d_block(side, 1)
    res = pk.cg_partitioned(side, world, gs, config=pk.SolverConfig(max_iterations=400))
    assert_identical(res, oracle_run("cg", a, b, (geom.n_groups, geom.group_size), max_iterations=400))


def test_c4_partitioned_random_rhs_fixed_iterations(pk):
    side, gs = 16, 512
    geom = pk.slab_geometry(side, gs)
    a, _ = pk.gen_poisson3d_block(side, 1)
    b = np.random.default_rng(3).random(side ** 3)
    cfg = pk.SolverConfig(fixed_iterations=25, max_iterations=25)
    res = pk.cg_partitioned(side, 4, gs, b=b, config=cfg)
    assert_identical(res, oracle_run("cg", a, b, (geom.n_groups, geom.group_size), fixed=25, max_iterations=25))
    single = pk.cg_pipelined(a, b, config=cfg, context=geom)
    assert same(single.x, res.x) and same(single.residual_history, res.residual_history)


@pytest.mark.parametrize("n,k", [(3000, 5), (2000, 40), (600, 400)])
def test_matrix_market_unstructured_rows(pk, tmp_path, n, k):
    """Unstructured rows: the reference's random family
    written to / read from Matrix Market, rows of 5, 40 (several SpMV passes)
    and 400 entries; pipelined and classical drivers bitwise vs the oracle."""
    a0, b = pk.gen_random_rowwise(n, k, seed=k)
    path = tmp_path / "rand.mtx"
    pk.write_matrix_market(path, a0)
    a = pk.read_matrix_market(path)
    assert a.equals(a0)
    for method in ("bicgstab", "gmres"):
        res = pk.SOLVERS[(method, "pipelined")](a, b, config=pk.SolverConfig(max_iterations=60))
        assert_identical(res, oracle_run(method, a, b, (128, 256), max_iterations=60))
        res = pk.SOLVERS[(method, "classical")](a, b, config=pk.SolverConfig(max_iterations=60))
        assert_identical(res, orc.CLASSICAL[method](a, b, geom=(128, 256), max_iterations=60))


# ---------------------------------------------------------------------------
# SELL-32 storage: the same entries walked slot-major
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", [n for n in gd.solver_case_names()
                                  if any(k in n for k in ("p2", "random", "cd2", "cd3", "x0", "eye5"))])
def test_sell32_solvers_match_reference_golden(pk, name):
    """Every solver on the SELL-32 copy of the golden matrices is bit-identical
    to the reference (same entries, same per-row order)."""
    case = gd.solver_case(name)
    store = gd.solvers()
    a = pk.CsrMatrix(*gd.csr_arrays(store, f"{name}/A"))
    ctx = pk.ExecutionContext(*case["geom"])
    dm = pk.DeviceMatrix.upload(pk.context_for(ctx), a).set_format("sell32", ctx)
    assert dm.format == "sell32" and dm.stored_entries >= a.nnz
    res = pk.SOLVERS[(case["method"], "pipelined")](dm, store[f"{name}/b"], x0=store.get(f"{name}/x0"),
                                                    config=pk.SolverConfig(**case["config"]), context=ctx)
    assert res.iterations == case["iterations"] and res.termination == case["termination"]
    assert same(res.residual_history, store[f"{name}/history"])
    assert same(res.x, store[f"{name}/x"])
    assert res.true_final_residual == store[f"{name}/true_final_residual"][0]


@pytest.mark.parametrize("n,k", [(3000, 5), (2000, 40), (600, 400)])
@pytest.mark.parametrize("method", ["cg", "bicgstab"])
def test_sell32_unstructured_rows_equal_csr(pk, n, k, method):
    """Ragged slices (rows of k entries, padded to the slice maximum): the
    SELL-32 walk equals the CSR walk bit for bit, fused and split bodies."""
    a, b = pk.gen_random_rowwise(n, k, seed=5)
    ctx = pk.ExecutionContext(8, 64)
    cfg = pk.SolverConfig(fixed_iterations=12, max_iterations=12)
    r_csr = pk.SOLVERS[(method, "pipelined")](a, b, config=cfg, context=ctx)
    dm = pk.DeviceMatrix.upload(pk.context_for(ctx), a).set_format("sell32", ctx)
    r_sell = pk.SOLVERS[(method, "pipelined")](dm, b, config=cfg, context=ctx)
    assert same(r_csr.x, r_sell.x) and same(r_csr.residual_history, r_sell.residual_history)
    dm.set_format("csr", ctx)
    assert dm.format == "csr"


@pytest.mark.parametrize("m", [34, 40, 70])
def test_gmres_restart_longer_than_one_update_chunk(pk, m):
    """GMRES(m) with m - 1 > 32 basis vectors per update: the Gram-Schmidt
    accumulation runs in 32-vector chunks through an accumulator vector
    (OpGsAcc, then OpGsUpdate) -- the same rounding sequence as the
    reference's single accumulated sum (fused.py:268-272)."""
    a, b = pk.convdiff2d(24)
    cfg = pk.SolverConfig(restart=m, max_iterations=200)
    res = pk.gmres_pipelined(a, b, config=cfg)
    assert_identical(res, oracle_run("gmres", a, b, (128, 256), restart=m, max_iterations=200))
    cfgf = pk.SolverConfig(restart=m, fixed_iterations=m + 3, max_iterations=m + 3)
    resf = pk.gmres_pipelined(a, b, config=cfgf, context=pk.ExecutionContext(8, 32))
    assert_identical(resf, oracle_run("gmres", a, b, (8, 32), restart=m, fixed=m + 3, max_iterations=m + 3))


def test_cached_workspace_survives_scratch_growth(pk):
    """A cached workspace's graph holds the context's scratch pointers: a later
    solve on the same context that grows (reallocates) the VEC buffer (a long-
    row matrix) or the spill (GMRES: 32 lane chains per lane) must drop the
    cache -- the repeated CG solve is then rebuilt and still bit-identical to
    its first run and to the oracle."""
    ctx = pk.ExecutionContext(16, 64)
    a_small, b_small = pk.gen_poisson2d(4)  # 127^2 rows, 5 per row
    cfg = pk.SolverConfig(max_iterations=300)
    first = pk.cg_pipelined(a_small, b_small, config=cfg, context=ctx)
    big, bb = pk.gen_random_rowwise(60000, 20, seed=4)  # VEC rows (>= 12 per row on average)
    fixed3 = pk.SolverConfig(fixed_iterations=3, max_iterations=3)
    for grow in (lambda: pk.cg_pipelined(big, bb, config=fixed3, context=ctx),
                 lambda: pk.gmres_pipelined(a_small, b_small, config=pk.SolverConfig(fixed_iterations=3,
                                                                                   max_iterations=3, restart=30),
                                            context=ctx)):
        grow()
        again = pk.cg_pipelined(a_small, b_small, config=cfg, context=ctx)
        assert again.iterations == first.iterations
        assert same(again.x, first.x) and same(again.residual_history, first.residual_history)
    assert_identical(first, oracle_run("cg", a_small, b_small, (16, 64), max_iterations=300))


def test_cached_workspace_survives_format_change(pk):
    """Switching a device matrix between SELL-32 and CSR frees / builds the
    SELL copy that cached graphs may walk: the matrix takes a new identity,
    so the next solve builds a fresh workspace; results stay bit-identical."""
    from paper_1410_4054_b200.solvers import solve_resident

    ctx = pk.ExecutionContext(16, 64)
    dc = pk.context_for(ctx)
    a, b = pk.gen_random_rowwise(20000, 8, seed=2)
    dm = pk.DeviceMatrix.upload(dc, a)
    bt = torch.from_numpy(np.asarray(b)).cuda()
    cfg = pk.SolverConfig(fixed_iterations=20, max_iterations=20)
    runs = []
    for fmt in ("sell32", "csr", "sell32", "csr"):
        dm.set_format(fmt, ctx)
        x, r = solve_resident("cg", dm, bt, config=cfg, context=ctx)
        runs.append((x.cpu().numpy(), list(r.residual_history)))
    for x, h in runs[1:]:
        assert same(x, runs[0][0]) and same(h, runs[0][1])


@pytest.mark.parametrize("persist", ["0", "1"])
def test_bicgstab_persistent_loop_identical(pk, persist, monkeypatch):
    """The split BiCGStab loop as one persistent cooperative kernel (grid
    barriers between the phases) or as the WHILE graph: the same bits, the
    same iterations; launches per iteration 0 vs 3.  Runs to tolerance (the
    finalizers' STOPPING / half-step exits) on a 2^20-row system."""
    monkeypatch.setenv("PK_PERSIST", persist)
    dm, b = pk.convdiff2d(1024, device=True)
    a, _ = pk.convdiff2d(1024)
    cfg = pk.SolverConfig(fixed_iterations=24, max_iterations=24)
    res = pk.bicgstab_pipelined(dm, b, config=cfg)
    assert_identical(res, oracle_run("bicgstab", a, b, (128, 256), fixed=24, max_iterations=24))
    assert [p.launches for p in res.trace.iterations[:2]] == ([0, 0] if persist == "1" else [3, 3])
