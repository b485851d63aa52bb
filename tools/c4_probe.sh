mkdir -p gpurun_out/c4s
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c4s/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/c4s/tests.log
for sp in 0 1; do
PK_CG_SPLIT=$sp timeout 600 python bench.py --workload c4 --steps 30 --warmup 3 > gpurun_out/c4s/c4_512_split$sp.json 2>&1
PK_CG_SPLIT=$sp timeout 600 python bench.py --workload c4 --side 256 --steps 30 --warmup 3 > gpurun_out/c4s/c4_256_split$sp.json 2>&1
done
timeout 600 python bench.py --workload c1 --steps 30 > gpurun_out/c4s/c1.json 2>&1
timeout 900 python bench.py --workload c5 --nsys 192 > gpurun_out/c4s/c5.json 2>&1
