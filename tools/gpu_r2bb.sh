set -u
OUT=gpurun_out/r2bb; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" $OUT/tests.log | tail -2
