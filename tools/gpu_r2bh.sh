set -u
OUT=gpurun_out/r2bh; mkdir -p $OUT
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
for f in bench bench_default; do python -c "
import json; d=json.loads(open('$OUT/'+'$f'+'.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['roofline']['frac'], d['iteration_roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['c1']['us_per_iter'], d['c1']['vs_floor'], d['c3']['us_per_iter_inner'], d['clocks']['reasons'])"; done
