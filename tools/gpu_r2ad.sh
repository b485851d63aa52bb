set -u
OUT=gpurun_out/r2ad; mkdir -p $OUT
PK_MAT_DISCARD=0 bash tools/ncu_capture.sh $OUT/ncu_tiles "k_reduce_tiles" 30 2 bicgstab 16 host
