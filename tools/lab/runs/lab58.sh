# MrgSN row tiles with component 1 by the integer half-step on a subset of steps (mask over 4): alone and sustained
mkdir -p gpurun_out
B=tools/lab/build
for v in m0 m1 m5 m7 m15; do
  echo "$v alone $(timeout 120 $B/fill_lab $B/libshv_$v.so 20 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['mrg_u32']; print(v['ms_best'], v['ms_mean'], v['sum'], v['wxor'])")"
done 2>&1 | tee gpurun_out/lab58.txt
for r in 1 2; do for v in m0 m1 m5 m7 m15; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/power_lab.py alt 60)"; sleep 3; done; done 2>&1 | tee -a gpurun_out/lab58.txt
