B=tools/lab/build
for r in 1 2; do for m in 0 1 4 5 16 17 20 21 32 33 36 37 48 49 52 53; do
  echo "ck$m $(timeout 60 $B/fill_lab $B/libshv_ck$m.so 6 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['mrg_u32']; print(v['ms_best'], v['sum'])")"
done; done 2>&1 | tee gpurun_out/lab13.txt
