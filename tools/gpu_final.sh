#!/bin/bash
# Round-end measurement pass (one gpurun call): smoke, GPU tests, headline
# bench + reference arm, launch list, ncu of the loop kernels, other configs.
set -u
TAG=${1:-final}
OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_round.sh $TAG smoke tests bench launches ncu ncu_cg
timeout 900 python bench.py --workload c1 --steps 30 > $OUT/c1.json 2> $OUT/c1.err; echo "c1 rc=$?"
timeout 900 python bench.py --workload c3 --steps 300 --warmup 3 > $OUT/c3.json 2> $OUT/c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --workload c4 --steps 30 --warmup 3 > $OUT/c4_512.json 2> $OUT/c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --workload c4 --side 256 --steps 30 --warmup 3 > $OUT/c4_256.json 2>> $OUT/c4.err; echo "c4b rc=$?"
timeout 900 python bench.py --workload c5 --nsys 192 > $OUT/c5_192.json 2> $OUT/c5.err; echo "c5 rc=$?"
timeout 900 python tools/engine_probe.py bicgstab:1024:a bicgstab:2048:a cg:512:a cg3d:128:a cg3d:256:a gmres:128:a > $OUT/engine_probe.jsonl 2>&1; echo "probe rc=$?"
timeout 600 python tools/dbg_simple.py > $OUT/dbg_simple.txt 2>&1; echo "dbg rc=$?"
