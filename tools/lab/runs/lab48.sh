# MrgSN (subnormal-state step) in the row-tile fill and MC: alone timings vs MrgIF
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in if5 sn5 sn4 sn5s128 sn4s128; do
  echo "$v $(timeout 120 $B/fill_lab $B/libshv_$v.so 40 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['mrg_u32']; print(v['ms_best'], v['ms_mean'], v['sum'], v['wxor'])")"
  sleep 2
done; done 2>&1 | tee gpurun_out/lab48.txt
for v in if5 sn5; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 5)"; done 2>&1 | tee -a gpurun_out/lab48.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "mrg or rows or parity or mc" 2>&1 | tail -5 | tee -a gpurun_out/lab48.txt
