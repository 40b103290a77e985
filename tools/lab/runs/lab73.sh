# MrgMF row tiles at S = 64 / 128 / 256
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in cur ms64 ms256; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 20 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['mrg_u32']['ms_best'], d['mrg_u32']['ms_mean'], d['mrg_u32']['sum'])")"; done; done 2>&1 | tee gpurun_out/lab73.txt
