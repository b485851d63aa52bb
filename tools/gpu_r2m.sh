set -u
OUT=gpurun_out/r2m; mkdir -p $OUT
timeout 300 python tools/engine_probe.py gmres:128:a gmres:64:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
PK_LIB_VARIANT=ld4 timeout 300 python tools/engine_probe.py gmres:128:a gmres:64:a > $OUT/probe_ld4.jsonl 2>&1; cat $OUT/probe_ld4.jsonl
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -x -q -k "gmres or fused or kernels" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
