#!/bin/bash
# Round-end pass + on-box ncu summaries (the .ncu-rep files are dropped so the
# merged gpurun_out/ stays under the 64 MiB cap).
set -u
TAG=${1:-final}
OUT=gpurun_out/$TAG
bash tools/gpu_final.sh $TAG
python tools/ncu_summary.py $OUT/bicgstab_full.ncu-rep $OUT/ncu_bicgstab_loop --traffic > $OUT/ncu_sum.log 2>&1
python tools/ncu_summary.py $OUT/cg_full.ncu-rep $OUT/ncu_cg_loop >> $OUT/ncu_sum.log 2>&1
cp profiles/ncu_traffic.json $OUT/ncu_traffic.json
ncu -i $OUT/bicgstab_full.ncu-rep --page details --csv > $OUT/ncu_bicgstab_details.csv 2>/dev/null
rm -f $OUT/*.ncu-rep
du -sh $OUT
