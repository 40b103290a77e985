B=tools/lab/build
for r in 1 2; do for v in r2if4 r2ff4 r2if5 r2old; do
  echo "== $v $(timeout 60 $B/fill_lab $B/libshv_$v.so 10 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms_best'],v['GBps'],v['sum']) for k,v in d.items() if k in ('mrg_u32',)})")"
done; done 2>&1 | tee gpurun_out/lab6.txt
