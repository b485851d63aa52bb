set -u
export PK_LIB_VARIANT=ckpt
OUT=gpurun_out/r2ah; mkdir -p $OUT
timeout 300 python tools/e2e_profile.py > $OUT/e2e_profile.txt 2>&1; head -30 $OUT/e2e_profile.txt
timeout 600 python tools/engine_probe.py bicgstab:1024:a cg:512:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 600 $OUT/bench.json
