"""C5 transient batch timing (BASELINE configs[4]) on this GPU: nsys 2D
Poisson systems, sides cycling 128/256/512, RHS default_rng(s).random(n),
pipelined CG to tol 1e-8, solved with solve_batch(threads).  Prints JSON."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1410_4054_b200 as pk

nsys = int(sys.argv[1]) if len(sys.argv) > 1 else 96
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 16
mode = sys.argv[3] if len(sys.argv) > 3 else "graph"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
sides = [128, 256, 512]
mats = {s: pk.poisson2d_grid(s)[0] for s in sides}
systems = [(mats[sides[i % 3]], np.random.default_rng(i).random(sides[i % 3] ** 2)) for i in range(nsys)]
cfg = pk.SolverConfig(max_iterations=5000, loop_mode=mode)
pk.solve_batch(systems[:3], tag="cg", config=cfg, threads=3)  # upload + warm
walls = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = pk.solve_batch(systems, tag="cg", config=cfg, threads=threads)
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
wall = sorted(walls)[len(walls) // 2]
its = [r.iterations for r in out]
loops = sum(r.loop_seconds for r in out)
print(json.dumps({"nsys": nsys, "threads": threads, "mode": mode, "sum_loop_s": round(loops, 4), "wall_s": round(wall, 4), "systems_per_s": round(nsys / wall, 2), "per_rep": [round(nsys / w, 1) for w in walls],
                  "iterations": {str(s): sorted(set(its[i] for i in range(nsys) if sides[i % 3] == s)) for s in sides},
                  "all_converged": all(r.termination == "converged" for r in out),
                  "sum_iterations": int(sum(its)), "us_per_iteration_aggregate": round(wall / sum(its) * 1e6, 3)}))
