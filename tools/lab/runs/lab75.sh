# MRG MC (MrgMF + integer hit) with 3 / 6 / 12 / 24 samples per unrolled iteration
mkdir -p gpurun_out
for r in 1 2; do for v in mu12 mu3 mu6 mu24; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/mc_lab.py mrg 2 | tail -1)"; done; done 2>&1 | tee gpurun_out/lab75.txt
