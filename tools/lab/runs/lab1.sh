mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in ff4 if4 if3 if2 null4; do
  echo "== $v r$r"; timeout 120 $B/fill_lab $B/libshv_$v.so 10
done; done > gpurun_out/lab1_fill.txt 2>&1
timeout 300 $B/tma_store_lab > gpurun_out/lab1_tma.txt 2>&1
cat gpurun_out/lab1_fill.txt gpurun_out/lab1_tma.txt | cut -c1-2000
