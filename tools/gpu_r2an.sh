set -u
OUT=gpurun_out/r2an; mkdir -p $OUT
timeout 900 compute-sanitizer --tool racecheck python tools/san_case.py vec host > $OUT/racecheck_vec_host.txt 2>&1; echo "racecheck vec host rc=$?"; grep -v "^=========     " $OUT/racecheck_vec_host.txt | tail -3
PK_VEC_MINAVG=0 timeout 900 compute-sanitizer --tool racecheck python tools/san_case.py vec graph > $OUT/racecheck_novec_graph.txt 2>&1; echo "racecheck novec graph rc=$?"; grep -v "^=========     " $OUT/racecheck_novec_graph.txt | tail -3
