B=tools/lab/build
for r in 1 2; do for v in s256 s512 s1024; do
  echo "$v $(timeout 120 $B/fill_lab $B/libshv_$v.so 40 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['mrg_u32']; print(v['ms_best'], v['ms_mean'], v['sum'])")"
  sleep 3
done; done 2>&1 | tee gpurun_out/lab43.txt
