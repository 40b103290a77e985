bash tools/lab/with_lib.sh lns python tools/lab/leap_lab.py philox 4 | tail -2 | tee gpurun_out/lab23.txt
bash tools/lab/with_lib.sh rt5 python tools/lab/leap_lab.py philox 4 | tail -2 | tee -a gpurun_out/lab23.txt
