set -u
OUT=gpurun_out/r2ak; mkdir -p $OUT
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
bash tools/ncu_capture.sh $OUT/ncu_c2 "k_reduce|k_sweep" 30 3 bicgstab 16 host
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches.csv python bench.py --loop host --steps 20 --warmup 3 --no-cpu --no-sub > $OUT/launches.log 2>&1; echo "launches rc=$?"
timeout 600 python tools/e2e_profile.py > $OUT/e2e_profile.txt 2>&1; head -1 $OUT/e2e_profile.txt
