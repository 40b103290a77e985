# MrgMF in the fills without a row-tile split (stream-per-lane TMA, staged f64 vector, scalar): vmf vs FF (vff)
mkdir -p gpurun_out
for r in 1 2; do for v in vff vmf; do echo "== $v"; bash tools/lab/with_lib.sh $v python tools/lab/vec_lab.py; done; done 2>&1 | tee gpurun_out/lab77.txt
