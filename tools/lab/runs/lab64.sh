# transposed Leap Frog fills: box height 16 / 32 / 64 player rows, 4 vs 8 warps per block
mkdir -p gpurun_out
for r in 1 2; do for v in lr32 lr16 lr64 lw8; do for g in philox mrg; do echo "$v $g $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py $g 5 | awk '{print $4}' | tr '\n' ' ')"; done; done; done 2>&1 | tee gpurun_out/lab64.txt
