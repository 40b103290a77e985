#!/bin/bash
# Build libshv variants (SHV_MRG_STEP x SHV_MRG_STAGE) and the lab driver.
set -e
cd "$(dirname "$0")/../.."
OUT=tools/lab/build; mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
C=paper_1412_8266_b200/csrc; SRCS="$C/kernels_mrg.cu $C/kernels_philox.cu $C/kernels_threefry.cu $C/kernels_tinymt32.cu $C/kernels_leapfrog.cu $C/kernels_audit.cu $C/kernels_mtgp32.cu $C/shv_api.cpp"
for step in ${STEPS:-0 2}; do for stage in ${STAGES:-0 1}; do
  nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -I include \
    -DSHV_MRG_STEP=$step -DSHV_MRG_STAGE=$stage $EXTRA \
    -o $OUT/libshv_s${step}_g${stage}.so $SRCS &
done; done
nvcc $ARCH -O3 -std=c++17 -o $OUT/fill_lab tools/lab/fill_lab.cu -ldl &
wait
ls $OUT
