"""Generate golden fixtures by running the REAL reference package.

Run in the development container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/fused_golden.npz, tests/golden/solver_golden.npz,
tests/golden/classical_golden.npz and tests/golden/manifest.json
(``--classical``: only the classical-driver fixtures, merged into the
existing manifest).  The fixtures pin the oracle (oracle/pk_oracle.py)
and, transitively, the CUDA path.  Inputs are stored alongside outputs so the
GPU box (which has no reference and may have different RNG streams) replays
exactly the same problems.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
REF = os.environ.get("PK_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import pipekrylov as pk  # noqa: E402  (the reference, read-only)
from pipekrylov.fused import WITH_INPUT, WITH_RESULT  # noqa: E402

from oracle import pk_oracle as orc  # noqa: E402  (only for the conv-diff arrays)

GEOMS = [(1, 1), (2, 4), (4, 8), (3, 16), (8, 32), (128, 256)]


def to_ref(a):
    return pk.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.cols, a.vals)


def put_csr(store, key, a):
    store[f"{key}/rowptr"] = np.asarray(a.row_offsets)
    store[f"{key}/cols"] = np.asarray(a.col_indices)
    store[f"{key}/vals"] = np.asarray(a.values)
    store[f"{key}/shape"] = np.array([a.n_rows, a.n_cols])


def fused_cases(store, manifest):
    rng = np.random.default_rng(20260101)
    dense = rng.standard_normal((300, 300))
    dense[rng.random((300, 300)) > 0.03] = 0.0
    np.fill_diagonal(dense, 4.0)
    a = pk.CsrMatrix.from_dense(dense)
    put_csr(store, "A", a)
    n = a.n_rows
    vecs = {name: rng.standard_normal(n) for name in ("p", "w", "x", "r", "s", "ap", "as", "r0", "v", "b0", "b1", "b2")}
    for name, v in vecs.items():
        store[f"vec/{name}"] = v
    for gi, (ng, gs) in enumerate(GEOMS):
        ctx = pk.ExecutionContext(n_groups=ng, group_size=gs)
        key = f"g{gi}"
        q, part = pk.spmv_fused(a, vecs["p"], pk.FusedReductionRequest((WITH_INPUT, WITH_RESULT, vecs["w"])), ctx)
        store[f"{key}/spmv/q"], store[f"{key}/spmv/part"] = q, part.data
        x, r, p = vecs["x"].copy(), vecs["r"].copy(), vecs["p"].copy()
        part = pk.fused_cg_vector_update(x, r, p, vecs["ap"], 0.37, -0.8, ctx)
        store[f"{key}/cg/x"], store[f"{key}/cg/r"], store[f"{key}/cg/p"] = x, r, p
        store[f"{key}/cg/part"] = part.data
        rr0 = pk.reduce_stage1(vecs["r"] * vecs["r0"], ctx)
        apr = pk.reduce_stage1(vecs["ap"] * vecs["r0"], ctx)
        s, spart, alpha = pk.fused_bicgstab_s_update(vecs["r"], vecs["ap"], rr0, apr, ctx)
        store[f"{key}/bs/rr0"], store[f"{key}/bs/apr"] = rr0.data, apr.data
        store[f"{key}/bs/s"], store[f"{key}/bs/part"] = s, spart.data
        store[f"{key}/bs/alpha"] = np.array([alpha])
        x, r, p = vecs["x"].copy(), vecs["r"].copy(), vecs["p"].copy()
        part = pk.fused_bicgstab_xrp_update(x, r, p, vecs["s"], vecs["ap"], vecs["as"], 0.3, 1.7, -0.4, vecs["r0"], ctx)
        store[f"{key}/xrp/x"], store[f"{key}/xrp/r"], store[f"{key}/xrp/p"] = x, r, p
        store[f"{key}/xrp/part"] = part.data
        basis = [vecs["b0"], vecs["b1"], vecs["b2"]]
        gpart = pk.fused_gs_stage1(basis, vecs["v"], ctx)
        store[f"{key}/gs1/part"] = gpart.data
        v = vecs["v"].copy()
        coeffs, npart = pk.fused_gs_update(v, basis, gpart, ctx)
        store[f"{key}/gsu/coeffs"], store[f"{key}/gsu/v"], store[f"{key}/gsu/part"] = coeffs, v.copy(), npart.data
        nrm, xpart = pk.fused_gs_normalize(v, npart, vecs["r"], ctx)
        store[f"{key}/gsn/norm"], store[f"{key}/gsn/v"], store[f"{key}/gsn/part"] = np.array([nrm]), v, xpart.data
        store[f"{key}/dot"] = np.array([pk.dot(vecs["x"], vecs["r"], ctx)])
        store[f"{key}/spmv_plain"] = pk.spmv_csr(a, vecs["x"])
    manifest["fused_geoms"] = GEOMS


def solver_cases():
    """(name, method, A(ref CsrMatrix), b, x0, config kwargs, geometry)."""
    cases = []
    p1, b1 = pk.gen_poisson2d(1)
    p2, b2 = pk.gen_poisson2d(2)
    rnd, brnd = pk.gen_random_rowwise(2000, 5, seed=3)
    cd2 = to_ref(orc.convdiff2d(24)[0])
    cd3 = to_ref(orc.convdiff3d(10)[0])
    spd = pk.CsrMatrix.from_dense([[4.0, 1.0], [1.0, 3.0]])
    upper = pk.CsrMatrix.from_dense([[2.0, 1.0], [0.0, 3.0]])
    sing = pk.CsrMatrix.from_dense([[1.0, 0.0], [0.0, 0.0]])
    eye = pk.CsrMatrix.identity(5)
    x0 = np.random.default_rng(7).standard_normal(p1.n_rows)
    rhs_rand = np.random.default_rng(11).random(p2.n_rows)
    for m in ("cg", "bicgstab", "gmres"):
        cases += [
            (f"{m}_p1", m, p1, b1, None, {}, (128, 256)),
            (f"{m}_p2", m, p2, b2, None, {}, (128, 256)),
            (f"{m}_p2_g4x64", m, p2, b2, None, {}, (4, 64)),
            (f"{m}_p2_g16x32", m, p2, b2, None, {}, (16, 32)),
            (f"{m}_p2_g1x1024", m, p2, b2, None, {}, (1, 1024)),
            (f"{m}_p2_randrhs", m, p2, rhs_rand, None, {}, (128, 256)),
            (f"{m}_p1_fixed30", m, p1, b1, None, {"fixed_iterations": 30, "max_iterations": 30}, (128, 256)),
            (f"{m}_p1_x0", m, p1, b1, x0, {}, (128, 256)),
            (f"{m}_p1_maxit7", m, p1, b1, None, {"max_iterations": 7}, (128, 256)),
            (f"{m}_zero_rhs", m, spd, np.zeros(2), None, {}, (128, 256)),
            (f"{m}_eye5", m, eye, np.arange(1.0, 6.0), None, {}, (128, 256)),
            (f"{m}_singular", m, sing, np.ones(2), None, {"max_iterations": 10}, (128, 256)),
        ]
    cases += [
        ("cg_spd2x2", "cg", spd, np.array([1.0, 2.0]), None, {"tolerance": 1e-12}, (128, 256)),
        ("bicgstab_upper2x2", "bicgstab", upper, np.array([3.0, 3.0]), None, {}, (128, 256)),
        ("gmres_upper2x2", "gmres", upper, np.array([3.0, 3.0]), None, {"tolerance": 1e-12}, (128, 256)),
        ("bicgstab_random", "bicgstab", rnd, brnd, None, {}, (128, 256)),
        ("gmres_random", "gmres", rnd, brnd, None, {}, (128, 256)),
        ("cg_random", "cg", rnd, brnd, None, {}, (128, 256)),
        ("bicgstab_cd2", "bicgstab", cd2, np.ones(cd2.n_rows), None, {}, (128, 256)),
        ("bicgstab_cd2_g8x32", "bicgstab", cd2, np.ones(cd2.n_rows), None, {}, (8, 32)),
        ("gmres_cd3", "gmres", cd3, np.ones(cd3.n_rows), None, {}, (128, 256)),
        ("gmres_cd2_m5", "gmres", cd2, np.ones(cd2.n_rows), None, {"restart": 5, "max_iterations": 200}, (128, 256)),
        ("gmres_cd3_fixed40", "gmres", cd3, np.ones(cd3.n_rows), None, {"fixed_iterations": 40, "max_iterations": 40}, (128, 256)),
        ("bicgstab_cd2_fixed25", "bicgstab", cd2, np.ones(cd2.n_rows), None, {"fixed_iterations": 25, "max_iterations": 25}, (128, 256)),
    ]
    return cases


def classical_cases():
    """The solver cases again through the reference's CLASSICAL drivers
    (solvers.py:310-389, 485-580, 725-858), plus modified Gram-Schmidt GMRES."""
    cases = [c for c in solver_cases() if "x0" in c[0] or "_p1" in c[0] or "_p2" in c[0] or "zero" in c[0]
             or "eye" in c[0] or "singular" in c[0] or "random" in c[0] or "cd2" in c[0] or "cd3" in c[0]
             or "2x2" in c[0]]
    p2, b2 = pk.gen_poisson2d(2)
    cd2 = to_ref(orc.convdiff2d(24)[0])
    cases += [
        ("gmres_p2_mgs", "gmres", p2, b2, None, {"orthogonalization": "modified_gs"}, (128, 256)),
        ("gmres_cd2_mgs_m7", "gmres", cd2, np.ones(cd2.n_rows), None,
         {"orthogonalization": "modified_gs", "restart": 7, "max_iterations": 150}, (16, 32)),
    ]
    return cases


def write_classical(manifest):
    store = {}
    manifest["classical_cases"] = []
    for name, method, a, b, x0, cfg, geom in classical_cases():
        fn = pk.SOLVERS[(method, "classical")]
        ctx = pk.ExecutionContext(n_groups=geom[0], group_size=geom[1])
        res = fn(a, b, x0=x0, config=pk.SolverConfig(**cfg), context=ctx)
        put_csr(store, f"{name}/A", a)
        store[f"{name}/b"] = np.asarray(b, dtype=np.float64)
        if x0 is not None:
            store[f"{name}/x0"] = np.asarray(x0, dtype=np.float64)
        store[f"{name}/x"] = res.x
        store[f"{name}/history"] = np.asarray(res.residual_history, dtype=np.float64)
        store[f"{name}/true_final_residual"] = np.array([res.true_final_residual])
        manifest["classical_cases"].append({
            "name": name, "method": method, "config": cfg, "geom": list(geom),
            "has_x0": x0 is not None, "iterations": res.iterations,
            "termination": res.termination, "breakdown_kind": res.breakdown_kind,
        })
        print(f"classical {name:24s} {res.termination:16s} it={res.iterations}")
    np.savez_compressed(HERE / "classical_golden.npz", **store)


def main():
    if "--classical" in sys.argv:
        # add the classical-driver fixtures without touching the others
        manifest = json.loads((HERE / "manifest.json").read_text())
        write_classical(manifest)
        (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1))
        return
    fused, manifest = {}, {}
    fused_cases(fused, manifest)
    np.savez_compressed(HERE / "fused_golden.npz", **fused)

    solvers = {}
    manifest["solver_cases"] = []
    for name, method, a, b, x0, cfg, geom in solver_cases():
        fn = pk.SOLVERS[(method, "pipelined")]
        ctx = pk.ExecutionContext(n_groups=geom[0], group_size=geom[1])
        res = fn(a, b, x0=x0, config=pk.SolverConfig(**cfg), context=ctx)
        put_csr(solvers, f"{name}/A", a)
        solvers[f"{name}/b"] = np.asarray(b, dtype=np.float64)
        if x0 is not None:
            solvers[f"{name}/x0"] = np.asarray(x0, dtype=np.float64)
        solvers[f"{name}/x"] = res.x
        solvers[f"{name}/history"] = np.asarray(res.residual_history, dtype=np.float64)
        solvers[f"{name}/true_final_residual"] = np.array([res.true_final_residual])
        manifest["solver_cases"].append({
            "name": name, "method": method, "config": cfg, "geom": list(geom),
            "has_x0": x0 is not None, "iterations": res.iterations,
            "termination": res.termination, "breakdown_kind": res.breakdown_kind,
            "launches_steady": [p.launches for p in res.trace.iterations[1:2]],
        })
        print(f"{name:24s} {res.termination:16s} it={res.iterations}")
    np.savez_compressed(HERE / "solver_golden.npz", **solvers)
    write_classical(manifest)
    manifest["reference"] = {"package": "pipekrylov", "version": pk.__version__,
                             "numpy": np.__version__}
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
