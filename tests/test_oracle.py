"""Pin the CPU oracle (oracle/pk_oracle.py) to the reference.

1. Against the committed golden fixtures produced by the real reference
   (tests/golden/make_golden.py) -- runs everywhere, bitwise.
2. Against the live reference when /root/reference is importable (dev
   container only) on extra cases, bitwise.
"""

import importlib
import sys

import numpy as np
import pytest

from oracle import pk_oracle as orc
from tests import golden_data as gd
from tests.conftest import REFERENCE_SRC, reference_available


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                                                 b.view(np.uint64) if b.dtype == np.float64 else b)


def golden_matrix():
    f = gd.fused()
    return orc.Csr(*gd.csr_arrays(f, "A"))


@pytest.mark.parametrize("gi", range(6))
def test_fused_ops_match_golden(gi):
    f = gd.fused()
    geom = tuple(gd.manifest()["fused_geoms"][gi])
    a = golden_matrix()
    v = {k.split("/")[1]: f[k] for k in f if k.startswith("vec/")}
    key = f"g{gi}"
    q, part = orc.spmv_fused(a, v["p"], ("input", "result", v["w"]), geom)
    assert same(q, f[f"{key}/spmv/q"]) and same(part, f[f"{key}/spmv/part"])
    assert same(orc.csr_spmv(a, v["x"]), f[f"{key}/spmv_plain"])

    x, r, p = v["x"].copy(), v["r"].copy(), v["p"].copy()
    part = orc.cg_update(x, r, p, v["ap"], 0.37, -0.8, geom)
    for name, arr in (("x", x), ("r", r), ("p", p), ("part", part)):
        assert same(arr, f[f"{key}/cg/{name}"]), name

    s, spart, alpha = orc.bicg_s_update(v["r"], v["ap"], f[f"{key}/bs/rr0"], f[f"{key}/bs/apr"], geom, 1e-30)
    assert same(orc.stage1(v["r"] * v["r0"], *geom), f[f"{key}/bs/rr0"])
    assert same(s, f[f"{key}/bs/s"]) and same(spart, f[f"{key}/bs/part"])
    assert alpha == f[f"{key}/bs/alpha"][0]

    x, r, p = v["x"].copy(), v["r"].copy(), v["p"].copy()
    part = orc.bicg_xrp_update(x, r, p, v["s"], v["ap"], v["as"], 0.3, 1.7, -0.4, v["r0"], geom)
    for name, arr in (("x", x), ("r", r), ("p", p), ("part", part)):
        assert same(arr, f[f"{key}/xrp/{name}"]), name

    basis = [v["b0"], v["b1"], v["b2"]]
    gpart = orc.gs_stage1(basis, v["v"], geom)
    assert same(gpart, f[f"{key}/gs1/part"])
    w = v["v"].copy()
    coeffs, npart = orc.gs_update(w, basis, gpart, geom)
    assert same(coeffs, f[f"{key}/gsu/coeffs"]) and same(w, f[f"{key}/gsu/v"])
    assert same(npart, f[f"{key}/gsu/part"])
    nrm, xpart = orc.gs_normalize(w, npart, v["r"], geom, 1e-30)
    assert nrm == f[f"{key}/gsn/norm"][0]
    assert same(w, f[f"{key}/gsn/v"]) and same(xpart, f[f"{key}/gsn/part"])
    assert orc.dot(v["x"], v["r"], geom) == f[f"{key}/dot"][0]


def run_oracle_case(case, store):
    name = case["name"]
    a = orc.Csr(*gd.csr_arrays(store, f"{name}/A"))
    b = store[f"{name}/b"]
    x0 = store.get(f"{name}/x0")
    cfg = case["config"]
    kw = dict(tol=cfg.get("tolerance", 1e-8), max_iterations=cfg.get("max_iterations", 500),
              fixed=cfg.get("fixed_iterations"), geom=tuple(case["geom"]))
    if case["method"] == "gmres":
        kw["restart"] = cfg.get("restart", 30)
    return orc.SOLVERS[case["method"]](a, b, x0=x0, **kw)


@pytest.mark.parametrize("name", gd.solver_case_names())
def test_solver_matches_golden(name):
    case = gd.solver_case(name)
    store = gd.solvers()
    res = run_oracle_case(case, store)
    assert res["iterations"] == case["iterations"]
    assert res["termination"] == case["termination"]
    assert res["breakdown_kind"] == case["breakdown_kind"]
    assert same(np.asarray(res["history"], dtype=np.float64), store[f"{name}/history"])
    assert same(res["x"], store[f"{name}/x"])
    assert res["true_final_residual"] == store[f"{name}/true_final_residual"][0]


def run_oracle_classical(case, store):
    name = case["name"]
    a = orc.Csr(*gd.csr_arrays(store, f"{name}/A"))
    b = store[f"{name}/b"]
    x0 = store.get(f"{name}/x0")
    cfg = case["config"]
    kw = dict(tol=cfg.get("tolerance", 1e-8), max_iterations=cfg.get("max_iterations", 500),
              fixed=cfg.get("fixed_iterations"), geom=tuple(case["geom"]))
    if case["method"] == "gmres":
        kw["restart"] = cfg.get("restart", 30)
        kw["mgs"] = cfg.get("orthogonalization") == "modified_gs"
    return orc.CLASSICAL[case["method"]](a, b, x0=x0, **kw)


@pytest.mark.parametrize("name", gd.classical_case_names())
def test_classical_matches_golden(name):
    """The oracle's classical drivers (solvers.py:310-389, 485-580, 725-858)
    reproduce the reference's own classical runs bitwise."""
    case = gd.classical_case(name)
    store = gd.classical()
    res = run_oracle_classical(case, store)
    assert res["iterations"] == case["iterations"]
    assert res["termination"] == case["termination"]
    assert res["breakdown_kind"] == case["breakdown_kind"]
    assert same(np.asarray(res["history"], dtype=np.float64), store[f"{name}/history"])
    assert same(res["x"], store[f"{name}/x"])
    assert res["true_final_residual"] == store[f"{name}/true_final_residual"][0]


def test_generators_match_reference_formulas():
    a, b = orc.poisson2d(1)
    assert a.n_rows == 225 and a.nnz == 1065  # test_io.py:180-189 KAT
    assert np.array_equal(b, np.ones(225))
    # the golden p1 case stores the reference's own gen_poisson2d(1) arrays
    _, _, rp, cols, vals = gd.csr_arrays(gd.solvers(), "cg_p1/A")
    assert same(a.rowptr, rp) and same(a.cols, cols) and same(a.vals, vals)
    _, _, rp, cols, vals = gd.csr_arrays(gd.solvers(), "cg_p2/A")
    a2, _ = orc.poisson2d(2)
    assert same(a2.rowptr, rp) and same(a2.cols, cols) and same(a2.vals, vals)


def test_stage1_known_answer():
    # test_linalg.py:145-152: 1024 ones at 4x256 -> partials [256]*4
    part = orc.stage1(np.ones(1024), 4, 256)
    assert np.array_equal(part[:, 0], [256.0] * 4)


# ---------------------------------------------------------------------------
# live reference (dev container only)
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def ref():
    if not reference_available():
        pytest.skip("reference not importable here")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    return importlib.import_module("pipekrylov")


@pytest.mark.reference
@pytest.mark.parametrize("side,block", [(8, 1), (12, 1), (9, 2)])
def test_poisson3d_matches_live_reference(ref, side, block):
    ra, _ = ref.gen_poisson3d_block(side, block)
    oa, _ = orc.poisson3d(side) if block == 1 else orc.poisson3d_block(side, block)
    assert same(ra.row_offsets, oa.rowptr) and same(ra.col_indices, oa.cols) and same(ra.values, oa.vals)


@pytest.mark.reference
@pytest.mark.parametrize("method", ["cg", "bicgstab", "gmres"])
@pytest.mark.parametrize("geom", [(128, 256), (7, 64), (2, 2048)])
def test_solvers_match_live_reference(ref, method, geom):
    a, b = ref.gen_poisson2d(3)
    rhs = np.random.default_rng(5).random(a.n_rows)
    cfg = ref.SolverConfig(max_iterations=150)
    ctx = ref.ExecutionContext(n_groups=geom[0], group_size=geom[1])
    rr = ref.SOLVERS[(method, "pipelined")](a, rhs, config=cfg, context=ctx)
    oo = orc.SOLVERS[method](a, rhs, max_iterations=150, geom=geom)
    assert oo["iterations"] == rr.iterations and oo["termination"] == rr.termination
    assert same(np.asarray(oo["history"]), np.asarray(rr.residual_history))
    assert same(oo["x"], rr.x)
    assert oo["true_final_residual"] == rr.true_final_residual


@pytest.mark.reference
@pytest.mark.parametrize("method", ["cg", "bicgstab", "gmres"])
@pytest.mark.parametrize("geom", [(128, 256), (7, 64)])
def test_classical_match_live_reference(ref, method, geom):
    """Oracle classical drivers vs the live reference's classical drivers on a
    fresh random-RHS case (GMRES with CGS and MGS)."""
    a, _ = ref.gen_poisson2d(3)
    rhs = np.random.default_rng(8).random(a.n_rows)
    ctx = ref.ExecutionContext(n_groups=geom[0], group_size=geom[1])
    for mgs in ((False, True) if method == "gmres" else (False,)):
        kw = {"orthogonalization": "modified_gs"} if mgs else {}
        rr = ref.SOLVERS[(method, "classical")](a, rhs, config=ref.SolverConfig(max_iterations=120, **kw), context=ctx)
        okw = {"mgs": mgs} if method == "gmres" else {}
        oo = orc.CLASSICAL[method](a, rhs, max_iterations=120, geom=geom, **okw)
        assert oo["iterations"] == rr.iterations and oo["termination"] == rr.termination
        assert same(np.asarray(oo["history"]), np.asarray(rr.residual_history))
        assert same(oo["x"], rr.x)
        assert oo["true_final_residual"] == rr.true_final_residual


@pytest.mark.reference
@pytest.mark.parametrize("m", [34, 40, 70])
def test_gmres_long_restart_oracle_matches_live_reference(ref, m):
    """The oracle the GPU's GMRES(m > 33) is checked against, vs the live
    reference on the same conv-diff system (any restart length)."""
    a = orc.convdiff2d(24)[0]
    ra = ref.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.cols, a.vals)
    b = np.ones(a.n_rows)
    rr = ref.SOLVERS[("gmres", "pipelined")](ra, b, config=ref.SolverConfig(restart=m, max_iterations=200))
    oo = orc.SOLVERS["gmres"](a, b, restart=m, max_iterations=200, geom=(128, 256))
    assert oo["iterations"] == rr.iterations and oo["termination"] == rr.termination
    assert same(np.asarray(oo["history"]), np.asarray(rr.residual_history))
    assert same(oo["x"], rr.x)
