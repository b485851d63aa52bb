set -u
OUT=gpurun_out/r2bi; mkdir -p $OUT
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --clock-control none -k regex:"k_bicg_persist" -c 1 --csv --page raw python tools/profile_target.py bicgstab 16 graph > $OUT/ncu_persist.csv 2> $OUT/ncu_persist.err; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r2bi/ncu_persist.csv')))
hdr=None
for i,r in enumerate(rows):
    if r and r[0]=='ID': hdr=r; units=rows[i+1]; data=rows[i+2]; break
if hdr:
    for w in ['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','launch__grid_size','sm__warps_active.avg.pct_of_peak_sustained_active']:
        for j,h in enumerate(hdr):
            if h==w: print(w, units[j], data[j][:80])
PY
