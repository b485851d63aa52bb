set -u
OUT=gpurun_out/r2ax; mkdir -p $OUT
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print(d['value'], json.dumps(d.get('roofline_wide')))"; tail -3 $OUT/bench.err
