set -u
OUT=gpurun_out/r2g; mkdir -p $OUT
for v in "" nosplit nostaged oldpro; do
  PK_LIB_VARIANT=$v timeout 300 python tools/engine_probe.py bicgstab:1024:PK_STAGE=0 cg:512:PK_STAGE=0 cg3d:256:PK_STAGE=0 gmres:128:PK_STAGE=0 > $OUT/probe_$v.jsonl 2>&1; echo "== variant '$v'"; cat $OUT/probe_$v.jsonl
done
PK_STAGE=0 timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests.log
PK_STAGE=0 timeout 600 python -m pytest tests/test_gpu_reference_suite.py -q -s > $OUT/refsuite.log 2>&1; echo "refsuite rc=$?"; tail -30 $OUT/refsuite.log
