set -u
OUT=gpurun_out/r2aw; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_PDL=1 bicgstab:1024:PK_PDL=1,PK_BULK=0 bicgstab:1024:PK_BULK_PDL=1 cg:512:PK_PDL=1 cg:512:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
