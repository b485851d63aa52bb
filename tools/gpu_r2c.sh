set -u
OUT=gpurun_out/r2c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -s > $OUT/scale.log 2>&1; echo "scale rc=$?"; tail -5 $OUT/scale.log
for v in "" sp1 sp4; do
  PK_LIB_VARIANT=$v timeout 300 python tools/engine_probe.py bicgstab:1024:a cg3d:256:a > $OUT/probe_$v.jsonl 2>&1; echo "probe $v"; cat $OUT/probe_$v.jsonl
done
PK_SWEEP_SCALAR=1 timeout 300 python tools/engine_probe.py bicgstab:1024:PK_SWEEP_SCALAR=1 cg3d:256:PK_SWEEP_SCALAR=1 > $OUT/probe_scalar.jsonl 2>&1; cat $OUT/probe_scalar.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
