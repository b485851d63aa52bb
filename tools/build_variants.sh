#!/bin/bash
# Engine experiments: build libpk_b200_<name>.so with extra -D flags
# (select at run time with PK_LIB_VARIANT=<name>).  usage: build_variants.sh name:FLAGS ...
cd "$(dirname "$0")/../paper_1410_4054_b200/csrc" || exit 1
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
    -Xcompiler -fPIC,-ffp-contract=off,-pthread -I../../include -I. $defs -shared -o ../libpk_b200_$name.so pk_capi.cu &
done
wait
ls -la ../libpk_b200_*.so
