set -u
OUT=gpurun_out/r2ab; mkdir -p $OUT
timeout 600 python tools/engine_probe.py bicgstab:1024:a bicgstab:1024:PK_TILE_MINK=0 bicgstab:2048:a gmres:128:a gmres:128:PK_TILE_MINK=0 cg3d:256:a cg3d:256:PK_TILE_MINK=0 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -k "bicgstab or cg or spmv or fused or gmres" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
