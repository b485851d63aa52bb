set -u
OUT=gpurun_out/r2e; mkdir -p $OUT
timeout 400 python tools/engine_probe.py bicgstab:1024:PK_STAGE=1 bicgstab:1024:PK_STAGE=0 cg3d:256:PK_STAGE=1 cg3d:256:PK_STAGE=0 gmres:128:PK_STAGE=1 gmres:128:PK_STAGE=0 bicgstab:2048:PK_STAGE=1 bicgstab:2048:PK_STAGE=0 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
