#!/bin/bash
# ncu --set full of the MRG fill and MC kernels of lab builds: bash tools/lab/ncu_lab.sh TAG lib1 lib2 ...
TAG=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mrg_fill_vec|mrg_mc" -c 2 \
    -o gpurun_out/lab_${TAG}_$v tools/lab/build/fill_lab tools/lab/build/libshv_$v.so 1 > gpurun_out/lab_${TAG}_$v.log 2>&1
  tail -2 gpurun_out/lab_${TAG}_$v.log
done
ls gpurun_out
