set -u
OUT=gpurun_out/r2ap; mkdir -p $OUT
for env in "X=1" "PK_LANE_SPMV=0" "PK_LANE_SPMV=0 PK_WARP_K1=1" "PK_BATCH_SMS=37"; do
  env $env timeout 600 python bench.py --workload c5 --nsys 192 --no-cpu > $OUT/c5.json 2>/dev/null; echo "$env $(python -c "import json;d=json.loads(open('$OUT/c5.json').read().strip().splitlines()[-1]);print(d['value'], d['config']['batch_wall_s'], d['all_converged'])")"
done
