"""Engine experiment: per-kernel event times of the BiCGStab / CG loop kernels
for several PK_ENGINE_FLAGS (removed) settings (each in a fresh process, since the
flags are read when a context is created).  Prints one JSON line per run."""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys, torch
sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk
from paper_1410_4054_b200.solvers import solve_resident
method, side = sys.argv[1], int(sys.argv[2])
import os
geom = tuple(int(v) for v in os.environ.get("PK_GEOM", "128x256").split("x"))
ctx = pk.ExecutionContext(*geom, device=0)
if method == "bicgstab":
    dm, b = pk.convdiff2d(side, device=True, context=ctx)
elif method == "cg3d":
    dm, b = pk.poisson3d_grid(side, device=True, context=ctx); method = "cg"
elif method == "gmres":
    dm, b = pk.convdiff3d(side, device=True, context=ctx)
else:
    dm, b = pk.poisson2d_grid(side, device=True, context=ctx)
b = torch.from_numpy(b).cuda()
it = 100
cfg = pk.SolverConfig(fixed_iterations=it, max_iterations=it, loop_mode="host")
solve_resident(method, dm, b, config=cfg, context=ctx, profile=True)
_, r = solve_resident(method, dm, b, config=cfg, context=ctx, profile=True)
g = pk.SolverConfig(fixed_iterations=it, max_iterations=it)
solve_resident(method, dm, b, config=g, context=ctx)
_, rg = solve_resident(method, dm, b, config=g, context=ctx)
ks, kl = r.diagnostics["kernel_seconds"], r.diagnostics["kernel_launches"]
print(json.dumps({"method": method, "side": side, "graph_us_per_iter": rg.loop_seconds / it * 1e6,
                  "kernel_us": [round(s / max(c, 1) * 1e6, 2) for s, c in zip(ks, kl) if c]}))
'''

if __name__ == "__main__":
    runs = sys.argv[1:] or ["bicgstab:1024:0"]
    for spec in runs:
        method, side, tag = spec.split(":")
        env = dict(os.environ)
        for kv in tag.split(","):  # e.g. PK_MULTIDOT_CAP=16,PK_PDL=0
            if "=" in kv:
                k, v = kv.split("=", 1)
                env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD, method, side], capture_output=True, text=True, env=env)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr.strip()[-400:]
        print(f"{tag} {line}", flush=True)
