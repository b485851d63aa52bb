"""Small solves for compute-sanitizer runs: `bulk` (BiCGStab 64^2 at 4 x 32 --
K = 32: the BULK engine) or `vec` (CG on a 40-per-row random matrix: the VEC
row sums)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1410_4054_b200 as pk  # noqa: E402
from paper_1410_4054_b200.solvers import solve_resident  # noqa: E402

case = sys.argv[1]
if case == "bulk":
    ctx = pk.ExecutionContext(4, 32, device=0)
    dm, b = pk.convdiff2d(64, device=True, context=ctx)
    cfg = pk.SolverConfig(fixed_iterations=3, max_iterations=3, loop_mode="host")
    solve_resident("bicgstab", dm, torch.from_numpy(b).cuda(), config=cfg, context=ctx)
else:
    a, bb = pk.gen_random_rowwise(2000, 40, seed=1)
    mode = sys.argv[2] if len(sys.argv) > 2 else "graph"
    pk.cg_pipelined(a, bb, config=pk.SolverConfig(fixed_iterations=3, max_iterations=3, loop_mode=mode),
                    context=pk.ExecutionContext(16, 64))
torch.cuda.synchronize()
print("san ok", case)
