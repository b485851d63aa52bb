set -u
OUT=gpurun_out/r2i; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reduce" -s 40 -c 3 -o $OUT/cg_c1 python tools/profile_target.py cg 16 host > $OUT/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"; tail -2 $OUT/ncu_c1.log
timeout 600 python bench.py --workload c5 --nsys 192 > $OUT/c5_192.json 2> $OUT/c5.err; echo "c5 rc=$?"; cat $OUT/c5_192.json; tail -3 $OUT/c5.err
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 $OUT/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -5 $OUT/racecheck.log
