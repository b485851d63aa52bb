set -u
OUT=gpurun_out/r2ag; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_BULK_PDL=0 bicgstab:1024:PK_BULK=0 cg:512:a gmres:128:a cg3d:256:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
