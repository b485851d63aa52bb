#!/bin/bash
# One ncu --set full capture of the C2 loop kernels (2 launches each) with
# source correlation; the report comes back in gpurun_out/<tag>/.
# usage: gpurun -- bash tools/gpu_ncu.sh <tag> [regex] [skip] [count] [target args...]
set -u
TAG=${1:-ncu}; RX=${2:-"k_reduce|k_sweep"}; SKIP=${3:-30}; CNT=${4:-6}
shift 4 || true
ARGS=${*:-"bicgstab 16 host"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c $CNT \
  -o $OUT/prof python tools/profile_target.py $ARGS > $OUT/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 $OUT/ncu.log
