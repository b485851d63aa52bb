set -u
OUT=gpurun_out/r2bd; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -x -q -k "check_phase" -v > $OUT/tests.log 2>&1; echo "tests rc=$?"; grep -E "PASS|FAIL|passed|failed" $OUT/tests.log | tail -8
