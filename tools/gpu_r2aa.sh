set -u
OUT=gpurun_out/r2aa; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_LIB_VARIANT=late bicgstab:1024:PK_LIB_VARIANT=laterp > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
PK_LIB_VARIANT=latetr timeout 300 python tools/bulk_trace.py 1024 > $OUT/trace.json 2>&1; cat $OUT/trace.json
