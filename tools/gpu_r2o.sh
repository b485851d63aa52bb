set -u
OUT=gpurun_out/r2o; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reduce|k_sweep" -s 30 -c 6 -o $OUT/c2 python tools/profile_target.py bicgstab 16 host > $OUT/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"; tail -1 $OUT/ncu_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reduce" -s 140 -c 8 -o $OUT/gmres python tools/profile_target.py gmres 30 host > $OUT/ncu_gmres.log 2>&1; echo "ncu gmres rc=$?"; tail -1 $OUT/ncu_gmres.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reduce" -s 26 -c 2 -o $OUT/cg_c1 python tools/profile_target.py cg 16 host > $OUT/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"; tail -1 $OUT/ncu_c1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --loop host --steps 20 --warmup 3 --no-cpu --no-sub > $OUT/launches.log 2>&1; echo "launches rc=$?"
