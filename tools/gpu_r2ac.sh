set -u
OUT=gpurun_out/r2ac; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:PK_MAT_DISCARD=0 bicgstab:2048:PK_MAT_DISCARD=0 gmres:128:PK_MAT_DISCARD=0 cg3d:256:PK_MAT_DISCARD=0 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
