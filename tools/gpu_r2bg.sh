set -u
OUT=gpurun_out/r2bg; mkdir -p $OUT
timeout 600 python tools/engine_probe.py cg:512:a cg:512:PK_PERSIST=0 cg:128:a cg:128:PK_PERSIST=0 bicgstab:1024:a > $OUT/probe.jsonl 2>&1; cut -c1-120 $OUT/probe.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" $OUT/tests.log | tail -2
