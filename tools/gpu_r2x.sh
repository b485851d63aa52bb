set -u
OUT=gpurun_out/r2x; mkdir -p $OUT
timeout 600 ./tools/ubench_tma > $OUT/ubench_tma.jsonl 2>&1; cat $OUT/ubench_tma.jsonl | sort -t: -k8 | tail -5; wc -l $OUT/ubench_tma.jsonl
