B=tools/lab/build
for v in mcif0 mcif1 mcff0 mcff1; do
  echo "$v $(timeout 120 $B/fill_lab $B/libshv_$v.so 1 256 0 0 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['mrg_mc'])")"
done 2>&1 | tee gpurun_out/lab18.txt
