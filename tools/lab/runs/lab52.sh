# MrgSN lane starts in the subnormal representation (ln) vs the FP64-split lane start (lo); 5 vs 4 blocks per SM
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in ln lo; do for bps in 5 4; do
  echo "$v b$bps $(timeout 120 $B/fill_lab $B/libshv_$v.so 40 256 $bps 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['mrg_u32']; print(v['ms_best'], v['ms_mean'], v['sum'], v['wxor'])")"
  sleep 2
done; done; done 2>&1 | tee gpurun_out/lab52.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "rows or parity" 2>&1 | tail -2 | tee -a gpurun_out/lab52.txt
