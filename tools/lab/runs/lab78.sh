# MrgMF stream-per-lane / vector fills: TMA fill at 2 vs 4 blocks per SM; parity tests of the non-row paths
mkdir -p gpurun_out
for r in 1 2; do for v in vmf2 vmf4; do echo "== $v"; bash tools/lab/with_lib.sh $v python tools/lab/vec_lab.py; done; done 2>&1 | tee gpurun_out/lab78.txt
timeout 1200 python -m pytest tests -m gpu -q -x -k "parity or rows or device or mrg" 2>&1 | tail -1 | tee -a gpurun_out/lab78.txt
