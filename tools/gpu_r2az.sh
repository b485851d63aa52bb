set -u
OUT=gpurun_out/r2az; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_PERSIST=1 bicgstab:2048:a bicgstab:2048:PK_PERSIST=1 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
PK_PERSIST=1 timeout 1500 python -m pytest tests -m gpu -x -q -k "bicgstab" > $OUT/tests.log 2>&1; echo "persist tests rc=$?"; tail -3 $OUT/tests.log
