# Leap Frog Philox transposed fill: 32-bit key words (k32) vs the widened XORs (k64), alternating
mkdir -p gpurun_out
for r in 1 2 3; do for v in k32 k64; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py philox 8 | sort -t: -k2 | head -1)"; done; done 2>&1 | tee gpurun_out/lab56.txt
