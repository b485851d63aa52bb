set -u
OUT=gpurun_out/r2ay; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['c1']['us_per_iter'], json.dumps(d.get('roofline_wide')))"
timeout 600 python tools/engine_probe.py bicgstab:1024:a cg:512:a gmres:128:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
