"""Golden fixtures for the reference's debug=True diagnostics.

Run in the development container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_debug_golden.py

Runs the reference's pipelined drivers with debug=True (CG rr_direct / beta,
solvers.py:417-467; BiCGStab s_dot_r0star / s_norm / identity_rr / direct_rr /
r0star_norm, 606-673; GMRES ortho_offdiag, 895-997) and stores every list in
tests/golden/debug_golden.npz + debug_manifest.json.  The cases include the
acceptance test's criterion-3 run (test_acceptance.py:151-178), a BiCGStab run
that stops on the half step, one through the check phase, and GMRES cycles.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, os.environ.get("PK_REFERENCE_SRC", "/root/reference/pkg/src"))

import pipekrylov as pk  # noqa: E402  (the reference, read-only)

from oracle import pk_oracle as orc  # noqa: E402  (conv-diff arrays only)


def to_ref(a):
    return pk.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.cols, a.vals)


def cases():
    p1, b1 = pk.gen_poisson2d(1)
    cd2 = to_ref(orc.convdiff2d(24)[0])
    cd3 = to_ref(orc.convdiff3d(10)[0])
    spec = json.loads((HERE / "scale_check_spec.json").read_text())["bicgstab_check_resume"]
    chk = pk.CsrMatrix.from_dense(spec["dense"])
    fixed30 = {"fixed_iterations": 30, "max_iterations": 30}
    return [
        ("cg_p1_fixed30", "cg", p1, b1, fixed30, (128, 256)),
        ("bicgstab_p1_fixed30", "bicgstab", p1, b1, fixed30, (128, 256)),
        ("cg_p1_tol", "cg", p1, b1, {}, (128, 256)),
        ("bicgstab_cd2_tol", "bicgstab", cd2, np.ones(cd2.n_rows), {}, (8, 32)),
        ("bicgstab_check_resume", "bicgstab", chk, np.asarray(spec["b"]), spec["config"], (128, 256)),
        ("gmres_cd3_tol", "gmres", cd3, np.ones(cd3.n_rows), {}, (128, 256)),
        ("gmres_cd2_m5", "gmres", cd2, np.ones(cd2.n_rows), {"restart": 5, "max_iterations": 60}, (16, 32)),
    ]


def main():
    store, manifest = {}, {"cases": []}
    for name, method, a, b, cfg, geom in cases():
        res = pk.SOLVERS[(method, "pipelined")](a, b, config=pk.SolverConfig(**cfg),
                                                context=pk.ExecutionContext(*geom), debug=True)
        store[f"{name}/rowptr"], store[f"{name}/cols"] = np.asarray(a.row_offsets), np.asarray(a.col_indices)
        store[f"{name}/vals"], store[f"{name}/b"] = np.asarray(a.values), np.asarray(b, dtype=np.float64)
        scalars = {}
        for key, val in res.diagnostics.items():
            if isinstance(val, list):
                store[f"{name}/{key}"] = np.asarray(val, dtype=np.float64)
            else:
                scalars[key] = val
        manifest["cases"].append({"name": name, "method": method, "config": cfg, "geom": list(geom),
                                  "shape": [a.n_rows, a.n_cols], "iterations": res.iterations,
                                  "lists": sorted(k for k, v in res.diagnostics.items() if isinstance(v, list)),
                                  "scalars": scalars})
        print(name, res.iterations, res.termination, {k: (len(v) if isinstance(v, list) else v)
                                                       for k, v in res.diagnostics.items()})
    np.savez_compressed(HERE / "debug_golden.npz", **store)
    (HERE / "debug_manifest.json").write_text(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
