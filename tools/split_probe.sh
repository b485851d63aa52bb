mkdir -p gpurun_out/split
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/split/tests3.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/split/tests3.log
PK_CG_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_solvers.py -x -q -k "golden or medium or loop_modes or unroll or c1 or batch" > gpurun_out/split/tests_cg.log 2>&1; echo tests_cg rc=$?; tail -2 gpurun_out/split/tests_cg.log
S=""
for rep in 1 2; do for t in PK_CG_SPLIT=0 PK_CG_SPLIT=1; do for w in cg:512 cg:1024 cg3d:128 cg3d:256; do S="$S $w:$t"; done; done; done
timeout 1200 python tools/engine_probe.py $S > gpurun_out/split/probe_cg.txt 2>&1
timeout 900 python bench.py > gpurun_out/split/bench.json 2> gpurun_out/split/bench.err; echo bench rc=$?
