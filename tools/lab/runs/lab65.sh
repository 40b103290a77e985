# magic-free subnormal quotients (k_sub = mul.rm(p_sub, inv) = D(k)): compute-only variants; MrgMF row tiles + MC alone and sustained
mkdir -p gpurun_out
B=tools/lab/build
timeout 120 $B/step4_lab > gpurun_out/lab65_step4.txt 2>&1; cat gpurun_out/lab65_step4.txt
for v in cur mf; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 10)"; done 2>&1 | tee gpurun_out/lab65.txt
for r in 1 2; do for v in cur mf; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/power_lab.py alt 60)"; sleep 3; done; done 2>&1 | tee -a gpurun_out/lab65.txt
