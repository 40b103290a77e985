# MrgSN row tiles after the register fixes (constant-memory multiplicands, pinned groups of 4)
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in if5 t128 t256 t128p1 t128np t64 t128m4; do
  echo "$v $(timeout 120 $B/fill_lab $B/libshv_$v.so 40 256 0 1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['mrg_u32']; print(v['ms_best'], v['ms_mean'], v['sum'], v['wxor'])")"
  sleep 2
done; done 2>&1 | tee gpurun_out/lab50.txt
echo "t128 $(timeout 200 $B/fill_lab $B/libshv_t128.so 5)" | tee -a gpurun_out/lab50.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mrg_fill_rows" -s 1 -c 1 \
    -o gpurun_out/lab50_t128 $B/fill_lab $B/libshv_t128.so 1 256 0 1 > gpurun_out/lab50_ncu.log 2>&1; tail -1 gpurun_out/lab50_ncu.log
