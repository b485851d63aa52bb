set -u
OUT=gpurun_out/r2q; mkdir -p $OUT
timeout 300 python tools/engine_probe.py gmres:128:a gmres:128:PK_GS_SPLIT=0 gmres:64:a gmres:64:PK_GS_SPLIT=0 > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
bash tools/ncu_capture.sh $OUT/ncu_c2 "k_reduce|k_sweep" 30 3 bicgstab 16 host
bash tools/ncu_capture.sh $OUT/ncu_gmres "k_reduce|k_sweep" 150 6 gmres 30 host
bash tools/ncu_capture.sh $OUT/ncu_c1 "k_reduce" 26 1 cg 16 host
du -sh $OUT
