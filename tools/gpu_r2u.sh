set -u
OUT=gpurun_out/r2u; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_BULK=0 bicgstab:2048:a bicgstab:2048:PK_BULK=0 cg3d:256:a cg3d:256:PK_BULK=0 gmres:128:a gmres:128:PK_BULK=0 cg:512:PK_BULK_MINK=2,PK_LANE_SPMV=0 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -k "bicgstab or cg or spmv or fused" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
bash tools/ncu_capture.sh $OUT/ncu_bulk "k_reduce" 30 2 bicgstab 16 host
