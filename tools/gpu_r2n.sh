set -u
OUT=gpurun_out/r2n; mkdir -p $OUT
for v in "" lp1 lp3; do
  PK_LIB_VARIANT=$v timeout 300 python tools/engine_probe.py bicgstab:1024:a bicgstab:2048:a cg:512:a cg:128:a gmres:128:a > $OUT/probe_$v.jsonl 2>&1; echo "== '$v'"; cat $OUT/probe_$v.jsonl
done
timeout 300 python tools/engine_probe.py bicgstab:1024:PK_LANE_SPMV=0 bicgstab:2048:PK_LANE_SPMV=0 cg:512:PK_LANE_SPMV=0 cg:128:PK_LANE_SPMV=0 gmres:128:PK_LANE_SPMV=0 > $OUT/probe_off.jsonl 2>&1; echo "== off"; cat $OUT/probe_off.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
