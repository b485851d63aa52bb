set -u
OUT=gpurun_out/r2ai; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 600 python tools/format_probe.py > $OUT/format_vec.jsonl 2>&1; cat $OUT/format_vec.jsonl
PK_VEC_MINAVG=0 timeout 600 python tools/format_probe.py > $OUT/format_novec.jsonl 2>&1; cat $OUT/format_novec.jsonl
timeout 300 python tools/e2e_profile.py > $OUT/e2e_profile.txt 2>&1; head -3 $OUT/e2e_profile.txt
cat > /tmp/san2.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk
from paper_1410_4054_b200.solvers import solve_resident
ctx = pk.ExecutionContext(4, 32, device=0)
dm, b = pk.convdiff2d(64, device=True, context=ctx)
b = torch.from_numpy(b).cuda()
cfg = pk.SolverConfig(fixed_iterations=5, max_iterations=5, loop_mode="host")
solve_resident("bicgstab", dm, b, config=cfg, context=ctx)
a, bb = pk.gen_random_rowwise(3000, 40, seed=1)
pk.cg_pipelined(a, bb, config=pk.SolverConfig(fixed_iterations=3, max_iterations=3), context=pk.ExecutionContext(16, 64))
torch.cuda.synchronize(); print("san ok")
PY
timeout 600 compute-sanitizer --tool memcheck python /tmp/san2.py > $OUT/memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -2 $OUT/memcheck.txt
timeout 600 compute-sanitizer --tool racecheck python /tmp/san2.py > $OUT/racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -2 $OUT/racecheck.txt
