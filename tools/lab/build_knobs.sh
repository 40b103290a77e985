#!/bin/bash
# Build libshv variants over the MRG fill knobs: name:flags pairs.
set -e
cd "$(dirname "$0")/../.."
OUT=tools/lab/build; mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
C=paper_1412_8266_b200/csrc; SRCS="$C/kernels_mrg.cu $C/kernels_philox.cu $C/kernels_threefry.cu $C/kernels_tinymt32.cu $C/kernels_leapfrog.cu $C/kernels_audit.cu $C/kernels_mtgp32.cu $C/shv_api.cpp"
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -I include $flags \
    -o $OUT/libshv_$name.so $SRCS &
done
wait
