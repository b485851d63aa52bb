#!/bin/bash
# two-phase engine A/B: per-kernel loop times with PK_MAT_MINK=0 (fused CTA
# engine) vs the default (two-phase for chains K >= 9), then GPU tests.
set -u
OUT=gpurun_out/${1:-mat}; mkdir -p $OUT
timeout 900 python tools/engine_probe.py bicgstab:1024:PK_MAT_MINK=0 bicgstab:1024:x bicgstab:2048:PK_MAT_MINK=0 bicgstab:2048:x \
  cg3d:256:PK_MAT_MINK=0 cg3d:256:x cg:512:PK_MAT_MINK=0 cg:512:x cg:512:PK_MAT_MINK=4 gmres:128:PK_MAT_MINK=0 gmres:128:x > $OUT/probe.txt 2>&1
echo "probe rc=$?"; cat $OUT/probe.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1
echo "tests rc=$?"; tail -15 $OUT/tests.log
