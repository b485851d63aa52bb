set -u
OUT=gpurun_out/r2s; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_BULK=0 bicgstab:1024:PK_BULK_RS=4 bicgstab:2048:a bicgstab:2048:PK_BULK=0 cg3d:256:a cg3d:256:PK_BULK=0 gmres:128:a gmres:128:PK_BULK=0 cg:512:PK_BULK_MINK=2,PK_LANE_SPMV=0 cg:512:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
cat > /tmp/san.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk
from paper_1410_4054_b200.solvers import solve_resident
ctx = pk.ExecutionContext(4, 32, device=0)
dm, b = pk.convdiff2d(64, device=True, context=ctx)
b = torch.from_numpy(b).cuda()
cfg = pk.SolverConfig(fixed_iterations=5, max_iterations=5, loop_mode="host")
solve_resident("bicgstab", dm, b, config=cfg, context=ctx)
torch.cuda.synchronize(); print("san ok")
PY
timeout 600 compute-sanitizer --tool memcheck python /tmp/san.py > $OUT/memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -3 $OUT/memcheck.txt
timeout 600 compute-sanitizer --tool racecheck python /tmp/san.py > $OUT/racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 $OUT/racecheck.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests.log
