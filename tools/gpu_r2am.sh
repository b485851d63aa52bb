set -u
OUT=gpurun_out/r2am; mkdir -p $OUT
for c in bulk vec; do
  timeout 900 compute-sanitizer --tool racecheck python tools/san_case.py $c > $OUT/racecheck_$c.txt 2>&1; echo "racecheck $c rc=$?"; grep -v "^=========     " $OUT/racecheck_$c.txt | tail -4
  timeout 900 compute-sanitizer --tool memcheck python tools/san_case.py $c > $OUT/memcheck_$c.txt 2>&1; echo "memcheck $c rc=$?"; tail -2 $OUT/memcheck_$c.txt
done
timeout 900 compute-sanitizer --tool synccheck python tools/san_case.py bulk > $OUT/synccheck_bulk.txt 2>&1; echo "synccheck rc=$?"; tail -2 $OUT/synccheck_bulk.txt
