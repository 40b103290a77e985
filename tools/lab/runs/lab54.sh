# MrgSI (component 1 integer, component 2 subnormal: 3 DFMA per number) vs MrgSN (6 DFMA): alone and sustained
mkdir -p gpurun_out
B=tools/lab/build
for v in cur si; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 10)"; done 2>&1 | tee gpurun_out/lab54.txt
for v in cur si; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/power_lab.py mrg 80)"; sleep 5; done 2>&1 | tee -a gpurun_out/lab54.txt
for v in cur si; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/power_lab.py alt 60)"; sleep 5; done 2>&1 | tee -a gpurun_out/lab54.txt
