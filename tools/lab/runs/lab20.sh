for g in philox threefry mrg; do python tools/lab/leap_lab.py $g 4; done 2>&1 | tee gpurun_out/lab20_leap.txt
timeout 900 python -m pytest tests/test_gpu_leapfrog.py -m gpu -q -x 2>&1 | tail -2 | tee -a gpurun_out/lab20_leap.txt
