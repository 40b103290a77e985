B=tools/lab/build
for r in 1 2; do for v in phl0 phl1; do
  echo "$v $(timeout 120 $B/fill_lab $B/libshv_$v.so 10 256 0 0 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:(v.get('ms_best', v.get('ms'))) for k,v in d.items() if k.startswith('philox')})")"
  bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py philox 4 | tail -1
done; done 2>&1 | tee gpurun_out/lab21.txt
