# MrgMF: magic-free lane starts (mfl) vs split_row_sn lane starts (mfl0); integer MC hit test (hi0)
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in mfl0 mfl hi0; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 20 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['mrg_u32']['ms_best'], d['mrg_u32']['ms_mean'], d['mrg_u32']['sum'], d['mrg_mc']['ms'], d['mrg_mc']['hits'])")"; done; done 2>&1 | tee gpurun_out/lab67.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "rows or parity or mc" 2>&1 | tail -2 | tee -a gpurun_out/lab67.txt
