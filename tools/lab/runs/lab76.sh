# Philox bulk fill with every round as IMAD + IMAD.HI (pa1) vs IMAD.WIDE (pa0): alone and alternating with MRG (power)
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in pa0 pa1; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 20 256 0 0 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['philox_u32']['ms_best'], d['philox_u32']['ms_mean'], d['philox_u32']['sum'])")"; done; done 2>&1 | tee gpurun_out/lab76.txt
for r in 1 2; do for v in pa0 pa1; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/power_lab.py alt 60)"; sleep 3; done; done 2>&1 | tee -a gpurun_out/lab76.txt
