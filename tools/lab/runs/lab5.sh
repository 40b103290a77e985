B=tools/lab/build
for v in rif4 rff4 ff4 rnull4; do for bps in 2 3 4; do
  echo "== $v bps$bps $(timeout 60 $B/fill_lab $B/libshv_$v.so 10 256 $bps 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms_best'],v['GBps']) for k,v in d.items() if k in ('mrg_u32','philox_u32')})")"
done; done 2>&1 | tee gpurun_out/lab5.txt
