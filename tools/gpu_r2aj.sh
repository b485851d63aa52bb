set -u
OUT=gpurun_out/r2aj; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "vec or long or mmio or unstructured or sell or spmv" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 600 python tools/format_probe.py > $OUT/format_vec.jsonl 2>&1; cat $OUT/format_vec.jsonl
