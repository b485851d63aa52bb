"""ncu target: a short fixed-iteration pipelined solve at a BASELINE config.

Usage: python tools/profile_target.py {bicgstab|cg|gmres} [iters] [loop_mode]

Runs one warm-up solve and one profiled solve on cuda:0 with inputs resident
in HBM, so `ncu -k regex:... -s <skip> -c <count>` can pick steady-state
launches of the fused kernels.  Not a bench (numbers under ncu are never
bench values)."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1410_4054_b200 as pk  # noqa: E402
from paper_1410_4054_b200.solvers import solve_resident  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "bicgstab"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 16
mode = sys.argv[3] if len(sys.argv) > 3 else "host"
geom = (128, 256)
ctx = pk.ExecutionContext(*geom, device=0)
if method == "bicgstab":
    dm, b = pk.convdiff2d(1024, device=True, context=ctx)
elif method == "cg":
    dm, b = pk.poisson2d_grid(512, device=True, context=ctx)
elif method == "cg3d":
    method = "cg"
    dm, b = pk.poisson3d_grid(256, device=True, context=ctx)
else:
    dm, b = pk.convdiff3d(128, device=True, context=ctx)
b = torch.from_numpy(b).cuda()
cfg = pk.SolverConfig(fixed_iterations=iters, max_iterations=iters, loop_mode=mode)
solve_resident(method, dm, b, config=cfg, context=ctx)
torch.cuda.synchronize()
_, res = solve_resident(method, dm, b, config=cfg, context=ctx)
torch.cuda.synchronize()
print(method, dm.n_rows, dm.nnz, res.iterations, res.termination, f"{res.loop_seconds / iters * 1e6:.2f} us/iter")
