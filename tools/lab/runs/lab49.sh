# MrgSN row tiles: S = 64 / 128 / 256, double-buffered boxes; ncu of IF S=256, SN S=128, SN S=256
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in sn5s64 sn5s128 sn5nb2 sn5; do
  echo "$v $(timeout 120 $B/fill_lab $B/libshv_$v.so 40 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['mrg_u32']; print(v['ms_best'], v['ms_mean'], v['sum'], v['wxor'])")"
  sleep 2
done; done 2>&1 | tee gpurun_out/lab49.txt
for v in if5 sn5s128 sn5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mrg_fill_rows" -s 1 -c 1 \
    -o gpurun_out/lab49_$v $B/fill_lab $B/libshv_$v.so 1 256 0 1 > gpurun_out/lab49_ncu_$v.log 2>&1
  tail -1 gpurun_out/lab49_ncu_$v.log
done
