# row tiles S = 128 (cur) vs S = 256 at 3/4/5 blocks per SM (in-flight tile footprint vs the L2): alone, 40 launches
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in cur t256; do for bps in 5 4 3; do
  echo "$v b$bps $(timeout 120 $B/fill_lab $B/libshv_$v.so 40 256 $bps 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['mrg_u32']; print(v['ms_best'], v['ms_mean'], v['sum'])")"
done; done; done 2>&1 | tee gpurun_out/lab59.txt
