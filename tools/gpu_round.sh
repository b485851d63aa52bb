#!/bin/bash
# One gpurun call: tests, bench, launch list and one full ncu capture.
# usage: gpurun -- bash tools/gpu_round.sh <tag> [what...]
#   what: tests bench launches ncu smoke (default: all)
set -u
TAG=${1:-r1}
shift || true
WHAT=${*:-"smoke tests bench launches ncu"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/nvsmi.txt" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1
for w in $WHAT; do
  case $w in
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
      echo "smoke rc=$?" ;;
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/tests.log" 2>&1
      echo "tests rc=$?"; tail -3 "$OUT/tests.log" ;;
    bench)
      timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
      echo "bench rc=$?"; tail -c 3000 "$OUT/bench.json"
      timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
      echo "bench ref rc=$?"; tail -c 1500 "$OUT/bench_ref.json" ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file "$OUT/launches.csv" python bench.py --loop host --steps 20 --warmup 3 --no-cpu > "$OUT/launches.log" 2>&1
      echo "launches rc=$?" ;;
    ncu)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 50 -c 2 \
        -o "$OUT/bicgstab_full" python tools/profile_target.py bicgstab 16 host > "$OUT/ncu.log" 2>&1
      echo "ncu rc=$?"; tail -3 "$OUT/ncu.log" ;;
    ncu_cg)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 25 -c 2 \
        -o "$OUT/cg_full" python tools/profile_target.py cg 16 host > "$OUT/ncu_cg.log" 2>&1
      echo "ncu_cg rc=$?"; tail -3 "$OUT/ncu_cg.log" ;;
    ncu_gmres)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 130 -c 8 \
        -o "$OUT/gmres_full" python tools/profile_target.py gmres 30 host > "$OUT/ncu_gmres.log" 2>&1
      echo "ncu_gmres rc=$?"; tail -3 "$OUT/ncu_gmres.log" ;;
    *)
      echo "unknown step $w" ;;
  esac
done
