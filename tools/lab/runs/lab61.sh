# transposed Leap Frog MRG32k3a fill: MrgIF vs MrgSN, 8-value groups unrolled 1 vs 4 (whole box)
mkdir -p gpurun_out
for r in 1 2; do for v in lfi1 lfi4 lfs1 lfs4; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py mrg 6 | awk '{print $4}' | tr '\n' ' ')"; done; done 2>&1 | tee gpurun_out/lab61.txt
