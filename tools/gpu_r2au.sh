set -u
OUT=gpurun_out/r2au; mkdir -p $OUT
timeout 600 python tools/engine_probe.py gmres:128:a gmres:128:PK_MDQ=0 gmres:64:a gmres:64:PK_MDQ=0 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q -k "gmres or gs or multidot or golden or stage1" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
