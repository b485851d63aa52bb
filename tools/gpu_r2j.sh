set -u
OUT=gpurun_out/r2j; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reduce" -s 20 -c 3 -o $OUT/cg_c1 python tools/profile_target.py cg 16 host > $OUT/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"; tail -2 $OUT/ncu_c1.log
timeout 600 python tools/engine_probe.py gmres:128:a gmres:128:PK_MULTIDOT_CAP=8 gmres:128:PK_MULTIDOT_CAP=4 gmres:128:PK_GS_CHUNK=16 gmres:128:PK_GS_CHUNK=8 gmres:128:PK_GS_CHUNK=8,PK_MULTIDOT_CAP=8 gmres:128:PK_GS_CHUNK=4,PK_MULTIDOT_CAP=4 > $OUT/gmres_probe.jsonl 2>&1; cat $OUT/gmres_probe.jsonl
