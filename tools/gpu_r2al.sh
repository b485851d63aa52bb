set -u
OUT=gpurun_out/r2al; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_BULK=0 cg:512:a gmres:128:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
