set -u
OUT=gpurun_out/r2ao; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:PK_BICG_SPLIT=0 bicgstab:1024:PK_BICG_SPLIT=0,PK_BULK=0 bicgstab:1024:a bicgstab:2048:a bicgstab:2048:PK_BICG_SPLIT=0 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
