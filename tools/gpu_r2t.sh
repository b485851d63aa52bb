set -u
OUT=gpurun_out/r2t; mkdir -p $OUT
bash tools/ncu_capture.sh $OUT/ncu_bulk "k_reduce" 30 2 bicgstab 16 host
