"""Golden fixtures at the BASELINE config sizes, produced by the REAL reference.

Run in the development container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_scale_golden.py [case ...]

Each case runs one pipelined driver of the reference (pipekrylov.SOLVERS,
__init__.py:81-88) on a config-sized system and stores, per case, in
tests/golden/scale/<case>.npz + tests/golden/scale_manifest.json:

* iterations, termination, breakdown kind, the full residual history and
  the true final residual;
* ``x_sha256``: SHA-256 of the solution's bytes -- the GPU test compares the
  WHOLE x bit for bit without committing megabytes;
* ``x_idx`` / ``x_sample``: x at 4096 fixed indices plus ``x_norm`` (for the
  relative-error comparison against a run at another reduction geometry).

The systems are the repo's pinned synthetic operators (oracle/pk_oracle.py
generators: gen_poisson3d_block(side, 1) arrays, the upwind
convection-diffusion operators the reference lacks), handed to the reference
as its own CsrMatrix.  Cases (VERDICT r1 "next" item 1):

  c4_128_tol_slab     CG 3D Poisson 128^3 to tol 1e-8, slab geometry 512 x 4096
  c4_128_tol_default  the same at the reference default geometry 128 x 256
  c4_256_fixed30_slab CG 3D Poisson 256^3, 30 fixed iterations, 256 x 65536
  c3_128_fixed31      GMRES(30) conv-diff 3D 128^3, 31 fixed steps (one full
                      cycle: trisolve, x update, restart), 128 x 256
  c3_64_tol / c3_128_tol  GMRES(30) conv-diff 3D to tol 1e-8 (cycle ends with the
                      true-residual gate), 128 x 256
  c2_1024_tol         BiCGStab conv-diff 2D 1024^2 to tol 1e-8, 128 x 256
  bicgstab_check_*    BiCGStab runs whose residual identity clamps to 0 below
                      tol, so the reference runs its "check" phase
                      (solvers.py:687-694): one passing, two failing + resuming
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE / "scale"
sys.path.insert(0, str(HERE.parents[1]))
REF = os.environ.get("PK_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import pipekrylov as pk  # noqa: E402  (the reference, read-only)

from oracle import pk_oracle as orc  # noqa: E402  (generator arrays only)

NSAMPLE = 4096


def to_ref(a):
    return pk.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.cols, a.vals)


def sample_idx(n):
    rng = np.random.default_rng(12345)
    return np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, NSAMPLE)])).astype(np.int64)


def check_system(name):
    """Small systems on which the BiCGStab residual identity goes negative
    while the monitor is below tol, so the reference runs its "check" phase
    (solvers.py:687-694): a 2x2 Jordan block whose first s is an exact
    eigenvector (check passes), and the same block plus three weakly excited
    modes at tol 1e-12 (check fails, the loop resumes, converges later).
    Found by a seeded search over such matrices; stored explicitly."""
    spec = json.loads((HERE / "scale_check_spec.json").read_text())[name]
    return pk.CsrMatrix.from_dense(spec["dense"]), np.asarray(spec["b"], dtype=np.float64), spec


CASES = {
    "c4_128_tol_slab": lambda: ("cg", to_ref(orc.poisson3d(128)[0]), None, {"max_iterations": 2000}, (512, 4096)),
    "c4_128_tol_default": lambda: ("cg", to_ref(orc.poisson3d(128)[0]), None, {"max_iterations": 2000}, (128, 256)),
    "c4_256_fixed30_slab": lambda: ("cg", to_ref(orc.poisson3d(256)[0]), None,
                                    {"fixed_iterations": 30, "max_iterations": 30}, (256, 65536)),
    "c3_128_fixed31": lambda: ("gmres", to_ref(orc.convdiff3d(128)[0]), None,
                               {"fixed_iterations": 31, "max_iterations": 31, "restart": 30}, (128, 256)),
    "c3_64_tol": lambda: ("gmres", to_ref(orc.convdiff3d(64)[0]), None, {"max_iterations": 3000, "restart": 30},
                          (128, 256)),
    "c3_128_tol": lambda: ("gmres", to_ref(orc.convdiff3d(128)[0]), None, {"max_iterations": 3000, "restart": 30},
                           (128, 256)),
    "c2_1024_tol": lambda: ("bicgstab", to_ref(orc.convdiff2d(1024)[0]), None, {"max_iterations": 20000},
                            (128, 256)),
}


def run_case(name):
    if name.startswith("bicgstab_check"):
        a, b, spec = check_system(name)
        method, cfg, geom = "bicgstab", spec["config"], tuple(spec["geom"])
    else:
        method, a, b, cfg, geom = CASES[name]()
    n = a.n_rows
    if b is None:
        b = np.ones(n)
    ctx = pk.ExecutionContext(n_groups=geom[0], group_size=geom[1])
    t0 = time.perf_counter()
    res = pk.SOLVERS[(method, "pipelined")](a, b, config=pk.SolverConfig(**cfg), context=ctx)
    wall = time.perf_counter() - t0
    idx = sample_idx(n)
    x = np.ascontiguousarray(res.x, dtype=np.float64)
    phases = [p.label for p in res.trace.phases]
    store = {
        "history": np.asarray(res.residual_history, dtype=np.float64),
        "true_final_residual": np.array([res.true_final_residual]),
        "x_idx": idx,
        "x_sample": x[idx],
        "x_norm": np.array([float(np.linalg.norm(x))]),
    }
    if n <= 20000:
        store["x"] = x
        store["b"] = np.asarray(b, dtype=np.float64)
    OUT.mkdir(exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **store)
    entry = {"name": name, "method": method, "n": n, "nnz": a.nnz, "config": cfg, "geom": list(geom),
             "iterations": res.iterations, "termination": res.termination, "breakdown_kind": res.breakdown_kind,
             "x_sha256": hashlib.sha256(x.tobytes()).hexdigest(), "check_phases": phases.count("check"),
             "reference_wall_s": round(wall, 2), "reference_loop_s_per_iter": res.loop_seconds / max(res.iterations, 1)}
    print(json.dumps(entry), flush=True)
    (OUT / f"{name}.json").write_text(json.dumps(entry, indent=1, sort_keys=True))
    return entry


def main(argv):
    if argv and argv[0] == "--merge":
        manifest = {"cases": {}, "reference": {"package": "pipekrylov", "version": pk.__version__,
                                               "numpy": np.__version__}}
        for f in sorted(OUT.glob("*.json")):
            manifest["cases"][f.stem] = json.loads(f.read_text())
        (HERE / "scale_manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True))
        return
    checks = list(json.loads((HERE / "scale_check_spec.json").read_text()))
    for name in argv or list(CASES) + checks:
        run_case(name)


if __name__ == "__main__":
    main(sys.argv[1:])
