# Leap Frog Philox run-to-run variance: same code (old = c816896, cur), every rep printed, fresh processes
mkdir -p gpurun_out
for r in 1 2 3; do for v in old cur; do echo "== $v"; bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py philox 8 | awk '{print $4}' | tr '\n' ' '; echo; done; done 2>&1 | tee gpurun_out/lab60.txt
