# transposed Leap Frog Philox with two t-columns per lane (256-B box rows) vs one
mkdir -p gpurun_out
for r in 1 2 3; do for v in cur pc2; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py philox 5 | awk '{print $4}' | tr '\n' ' ')"; done; done 2>&1 | tee gpurun_out/lab71.txt
bash tools/lab/with_lib.sh pc2 timeout 900 python -m pytest tests -m gpu -q -x -k "leap" 2>&1 | tail -2 | tee -a gpurun_out/lab71.txt
