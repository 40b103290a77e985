for r in 1 2; do for v in f128 f256; do echo "== $v"; bash tools/lab/with_lib.sh $v python tools/lab/sweep_lab.py; sleep 5; done; done 2>&1 | tee gpurun_out/lab45.txt
