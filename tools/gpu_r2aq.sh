set -u
OUT=gpurun_out/r2aq; mkdir -p $OUT
for rep in 1 2; do
for env in "X=1" "PK_BATCH_SMS=74" "PK_BATCH_SMS=37" "PK_BATCH_SMS=18" "PK_BATCH_SMS=9"; do
  env $env timeout 600 python bench.py --workload c5 --nsys 192 --no-cpu > $OUT/c5.json 2>/dev/null; echo "$env $(python -c "import json;d=json.loads(open('$OUT/c5.json').read().strip().splitlines()[-1]);print(d['value'], d['config']['batch_wall_s'], d['all_converged'])")"
done
done
