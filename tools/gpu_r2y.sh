set -u
OUT=gpurun_out/r2y; mkdir -p $OUT
timeout 600 ./tools/ubench_tma > $OUT/ubench_tma.jsonl 2>&1; wc -l $OUT/ubench_tma.jsonl
