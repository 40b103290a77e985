# transposed Leap Frog Philox / Threefry fills: 8-value groups unrolled 1 / 2 / 4
mkdir -p gpurun_out
for r in 1 2; do for v in lc1 lc2 lc4; do for g in philox threefry; do echo "$v $g $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py $g 5 | awk '{print $4}' | tr '\n' ' ')"; done; done; done 2>&1 | tee gpurun_out/lab62.txt
