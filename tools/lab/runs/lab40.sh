for g in tinymt mrg philox threefry; do python tools/lab/leap_lab.py $g 5 | tail -2; done 2>&1 | tee gpurun_out/lab40.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "leap or tinymt" 2>&1 | tail -2 | tee -a gpurun_out/lab40.txt
