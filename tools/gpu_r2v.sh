set -u
OUT=gpurun_out/r2v; mkdir -p $OUT
timeout 300 python tools/bulk_trace.py 1024 > $OUT/trace.json 2>&1; cat $OUT/trace.json
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_LIB_VARIANT=r4 bicgstab:1024:PK_LIB_VARIANT=w3 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
