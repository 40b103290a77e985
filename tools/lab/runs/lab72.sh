# MrgMF row tiles with the 48 / 64 / 85-register bounds (5 / 4 / 3 blocks per SM): alone and alternating with Philox
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in cur mb4 mb3; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 20 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['mrg_u32']['ms_best'], d['mrg_u32']['ms_mean'], d['mrg_u32']['sum'])")"; done; done 2>&1 | tee gpurun_out/lab72.txt
for v in cur mb4 mb3; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/power_lab.py alt 60)"; sleep 3; done 2>&1 | tee -a gpurun_out/lab72.txt
