set -u
OUT=gpurun_out/r2ar; mkdir -p $OUT
timeout 900 python tools/engine_probe.py gmres:128:a gmres:128:PK_LIB_VARIANT=dl32 gmres:128:PK_LIB_VARIANT=lt128 cg:512:PK_LIB_VARIANT=lt128 cg:512:a bicgstab:1024:PK_LIB_VARIANT=lt128 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
