set -u
OUT=gpurun_out/r2af; mkdir -p $OUT
PK_LIB_VARIANT=trace timeout 300 python tools/bulk_trace.py 1024 > $OUT/trace.json 2>&1; cat $OUT/trace.json
PK_LIB_VARIANT=trace timeout 300 python tools/engine_probe.py bicgstab:1024:PK_LIB_VARIANT=trace > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
