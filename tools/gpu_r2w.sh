set -u
OUT=gpurun_out/r2w; mkdir -p $OUT
./tools/ubench_chunk_order > $OUT/ubench.jsonl 2>&1; cat $OUT/ubench.jsonl
timeout 300 python tools/bulk_trace.py 1024 > $OUT/trace.json 2>&1; cat $OUT/trace.json
PK_LIB_VARIANT=tracenog timeout 300 python tools/bulk_trace.py 1024 > $OUT/trace_nog.json 2>&1; cat $OUT/trace_nog.json
