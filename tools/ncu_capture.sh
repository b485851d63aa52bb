#!/bin/bash
# ncu --set full capture on the GPU box, exported to small CSV/markdown files
# there (the .ncu-rep of this library exceeds gpurun's 64 MiB return limit).
# usage: bash tools/ncu_capture.sh <outdir> <regex> <skip> <count> <target args...>
set -u
OUT=$1; RX=$2; SKIP=$3; CNT=$4; shift 4
mkdir -p "$OUT"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s "$SKIP" -c "$CNT" \
  -o "$OUT/rep" python tools/profile_target.py "$@" > "$OUT/ncu.log" 2>&1
echo "ncu rc=$?"; tail -1 "$OUT/ncu.log"
ncu -i "$OUT/rep.ncu-rep" --page raw --csv > "$OUT/raw.csv" 2>/dev/null
ncu -i "$OUT/rep.ncu-rep" --page details --csv > "$OUT/details.csv" 2>/dev/null
ncu -i "$OUT/rep.ncu-rep" --page source --csv --print-source sass > "$OUT/source_sass.csv" 2>/dev/null
python tools/ncu_summary.py "$OUT/rep.ncu-rep" "$OUT/summary" > /dev/null 2>&1
python tools/stall_summary.py "$OUT/source_sass.csv" > "$OUT/stalls.md" 2>&1
gzip -f "$OUT/source_sass.csv" "$OUT/details.csv"
rm -f "$OUT/rep.ncu-rep"
ls -la "$OUT"
