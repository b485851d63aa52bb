set -u
OUT=gpurun_out/r2k; mkdir -p $OUT
timeout 400 python tools/engine_probe.py bicgstab:1024:a cg:512:a cg:128:a cg3d:256:a gmres:128:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 600 python bench.py --workload c4 --steps 30 --warmup 3 --no-cpu > $OUT/c4.json 2> $OUT/c4.err; echo "c4 rc=$?"; cat $OUT/c4.json; tail -3 $OUT/c4.err
PK_DCG_GRAPH=0 timeout 600 python bench.py --workload c4 --steps 30 --warmup 3 --no-cpu > $OUT/c4_nograph.json 2>> $OUT/c4.err; echo "c4ng rc=$?"; cat $OUT/c4_nograph.json
timeout 600 python bench.py --workload c4 --side 256 --steps 30 --warmup 3 --no-cpu > $OUT/c4_256.json 2>> $OUT/c4.err; cat $OUT/c4_256.json
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
