# Leap Frog Philox transposed fill with 32-bit key words (no widened XORs): C5 shape, then the Leap Frog GPU tests
mkdir -p gpurun_out
for r in 1 2; do for g in philox mrg threefry; do python tools/lab/leap_lab.py $g 6 | tail -1; done; done 2>&1 | tee gpurun_out/lab55.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "leap" 2>&1 | tail -2 | tee -a gpurun_out/lab55.txt
