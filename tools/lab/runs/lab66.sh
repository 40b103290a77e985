# MrgMF elsewhere: stream-per-lane / f64 vector fills (vmf vs FF default), transposed Leap Frog MRG (lmf unrolled, lmf1 not, vs IF)
mkdir -p gpurun_out
B=tools/lab/build
for v in cur vmf; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 10 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['mrg_u32']['ms_best'], d['mrg_f64']['ms_best'], d['mrg_f64']['sum'], d['mrg_mc']['ms'])")"; done 2>&1 | tee gpurun_out/lab66.txt
for r in 1 2; do for v in cur lmf lmf1; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py mrg 5 | awk '{print $4, $6}' | tr '\n' ' ')"; done; done 2>&1 | tee -a gpurun_out/lab66.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "mrg or rows or parity or mc or device" 2>&1 | tail -2 | tee -a gpurun_out/lab66.txt
