set -u
OUT=gpurun_out/r2p; mkdir -p $OUT
timeout 300 python tools/engine_probe.py gmres:128:a gmres:128:PK_GS_SPLIT=0 gmres:64:a cg:512:a bicgstab:1024:a > $OUT/probe.jsonl 2>&1; cat $OUT/probe.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -k "gmres or fused or kernels or golden" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reduce|k_sweep" -s 30 -c 3 -o $OUT/c2 python tools/profile_target.py bicgstab 16 host > $OUT/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"; tail -1 $OUT/ncu_c2.log
ls -la $OUT
