set -u
OUT=gpurun_out/r2l; mkdir -p $OUT
timeout 600 python tools/engine_probe.py gmres:128:a gmres:128:PK_LANE=0 gmres:64:a bicgstab:1024:a cg:512:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
