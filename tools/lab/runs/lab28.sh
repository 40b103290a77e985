for v in rt7 lt8; do for g in philox mrg threefry tinymt; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py $g 4 | tail -1)"; done; done 2>&1 | tee gpurun_out/lab28.txt
timeout 900 python -m pytest tests/test_gpu_leapfrog.py tests/test_gpu_tinymt.py -m gpu -q -x 2>&1 | tail -2 | tee -a gpurun_out/lab28.txt
