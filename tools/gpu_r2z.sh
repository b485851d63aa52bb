set -u
OUT=gpurun_out/r2z; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_LIB_VARIANT=rpldg bicgstab:1024:PK_BULK=0 gmres:128:PK_LIB_VARIANT=rpldg cg3d:256:PK_LIB_VARIANT=rpldg > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
PK_LIB_VARIANT=rpldgtr timeout 300 python tools/bulk_trace.py 1024 > $OUT/trace.json 2>&1; cat $OUT/trace.json
