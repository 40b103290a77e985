B=tools/lab/build
for r in 1 2; do for v in pm1 pm2; do
  echo "$v $(timeout 120 $B/fill_lab $B/libshv_$v.so 1 256 0 0 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['philox_mc'], d['mrg_mc'])")"
done; done 2>&1 | tee gpurun_out/lab38.txt
