# MRG32k3a f64 fill in row tiles (S = 64 doubles: 512-B segments) vs the staged vector kernel
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in f64v cur; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 20 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['mrg_f64']['ms_best'], d['mrg_f64']['ms_mean'], d['mrg_f64']['sum'], d['mrg_f64']['wxor'], d['mrg_u32']['ms_best'])")"; done; done 2>&1 | tee gpurun_out/lab70.txt
timeout 1500 python -m pytest tests -m gpu -q -x -k "rows or parity or f64 or device" 2>&1 | tail -2 | tee -a gpurun_out/lab70.txt
