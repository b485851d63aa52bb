set -u
OUT=gpurun_out/r2r; mkdir -p $OUT
timeout 300 python tools/engine_probe.py gmres:128:a gmres:128:PK_GS_SPLIT=0 gmres:64:a gmres:64:PK_GS_SPLIT=0 bicgstab:1024:a cg:512:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for t in 16 32; do timeout 600 python -c "
import sys, time, json; sys.path.insert(0, '.')
import numpy as np, torch, paper_1410_4054_b200 as pk
sides=[128,256,512]; mats={s: pk.poisson2d_grid(s)[0] for s in sides}
systems=[(mats[sides[i%3]], np.random.default_rng(i).random(sides[i%3]**2)) for i in range(192)]
cfg=pk.SolverConfig(max_iterations=5000)
pk.solve_batch(systems[:48], tag='cg', config=cfg, threads=$t)
torch.cuda.synchronize(); t0=time.perf_counter(); out=pk.solve_batch(systems, tag='cg', config=cfg, threads=$t); torch.cuda.synchronize()
print(json.dumps({'threads': $t, 'systems_per_s': 192/(time.perf_counter()-t0)}))
"; done
