"""Format experiment: CSR vs SELL-32 walk for short (stencil) and long
(unstructured, gen_random_rowwise) rows; per-iteration graph time of a
fixed-iteration pipelined solve, same bits either way.  CSR matrices with
>= PK_VEC_MINAVG entries per row (default 12) take the warp-cooperative VEC
row-sum pre-pass; run with PK_VEC_MINAVG=0 for thread-per-row CSR."""
import os
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk  # noqa: E402
from paper_1410_4054_b200.solvers import solve_resident  # noqa: E402
import torch  # noqa: E402

ctx = pk.ExecutionContext(128, 256)
dc = pk.context_for(ctx)
cases = [("random", 200000, 5), ("random", 200000, 40), ("random", 20000, 400), ("random", 1000000, 16)]
for fam, n, k in cases:
    a, b = pk.gen_random_rowwise(n, k, seed=1)
    for method in ("cg", "bicgstab"):
        out = {"matrix": f"{fam} n={n} k={k}", "method": method,
               "csr_walk": "vec" if k >= int(os.environ.get("PK_VEC_MINAVG", "12")) > 0 else "thread-per-row"}
        xs = {}
        for fmt in ("csr", "sell32"):
            dm = pk.DeviceMatrix.upload(dc, a).set_format(fmt, ctx)
            bt = torch.from_numpy(np.asarray(b)).cuda()
            it = 50
            cfg = pk.SolverConfig(fixed_iterations=it, max_iterations=it)
            solve_resident(method, dm, bt, config=cfg, context=ctx)
            x, r = solve_resident(method, dm, bt, config=cfg, context=ctx)
            out[fmt + "_us_per_iter"] = round(r.loop_seconds / it * 1e6, 2)
            xs[fmt] = x.cpu().numpy()
            dm.close()
        out["bitwise_equal"] = bool(np.array_equal(xs["csr"].view(np.uint64), xs["sell32"].view(np.uint64)))
        print(json.dumps(out), flush=True)
