#!/bin/bash
# usage: variant_probe.sh "v1 v2 ..." "method:side ..."  (PK_LIB_VARIANT builds from tools/build_variants.sh)
mkdir -p gpurun_out/var
S=""
for rep in 1 2; do for v in $1; do for w in $2; do S="$S $w:PK_LIB_VARIANT=$v"; done; done; done
timeout 1200 python tools/engine_probe.py $S > gpurun_out/var/probe.txt 2>&1
