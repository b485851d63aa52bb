mkdir -p gpurun_out/pdl
S=""
for rep in 1 2; do for t in PK_UNROLL=4 PK_UNROLL=8 PK_UNROLL=16; do for w in bicgstab:1024 cg:512 cg3d:128; do S="$S $w:$t"; done; done; done
timeout 1200 python tools/engine_probe.py $S > gpurun_out/pdl/probe2.txt 2>&1
