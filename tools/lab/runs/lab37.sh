B=tools/lab/build
for r in 1 2; do for v in gif mcu; do
  echo "$v $(timeout 120 $B/fill_lab $B/libshv_$v.so 1 256 0 0 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['mrg_mc'])")"
  sleep 3
done; done 2>&1 | tee gpurun_out/lab37.txt
timeout 600 python -m pytest tests -m gpu -q -x -k "mc" 2>&1 | tail -2 | tee -a gpurun_out/lab37.txt
