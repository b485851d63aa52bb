set -u
OUT=gpurun_out/r2ae; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:PK_TILE_MINK=9,PK_LIB_VARIANT=relaxed bicgstab:1024:PK_TILE_MINK=9,PK_LIB_VARIANT=tminb2 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
