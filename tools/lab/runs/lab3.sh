mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in rff4 rif4 rif3 rif2 rnull4 ff4; do
  echo "== $v r$r"; timeout 120 $B/fill_lab $B/libshv_$v.so 10 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms_best'],v['GBps'],v['sum']) for k,v in d.items() if k in ('mrg_u32',)})"
done; done 2>&1 | tee gpurun_out/lab3_fill.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/lab3_pytest.txt
