set -u
OUT=gpurun_out/r2as; mkdir -p $OUT
PK_VEC_MINAVG=12 timeout 900 python tools/format_probe.py > $OUT/format_vec12.jsonl 2>&1; cat $OUT/format_vec12.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
