set -u
OUT=gpurun_out/r2be; mkdir -p $OUT
for rep in 1 2; do
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_LIB_VARIANT=sleep0 bicgstab:1024:PK_LIB_VARIANT=sleep200 bicgstab:2048:a bicgstab:2048:PK_LIB_VARIANT=sleep0 bicgstab:2048:PK_LIB_VARIANT=sleep200 > $OUT/probe$rep.jsonl 2>&1; cut -c1-110 $OUT/probe$rep.jsonl
done
