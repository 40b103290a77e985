# sustained back-to-back fills with NVML clocks/power: current (MrgSN), MrgIF, null generator in the same row tiles; Philox; alternate
mkdir -p gpurun_out
for v in cur if5 nullrows; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/power_lab.py mrg 80)"; sleep 5; done 2>&1 | tee gpurun_out/lab53.txt
for p in philox alt; do echo "cur $(bash tools/lab/with_lib.sh cur python tools/lab/power_lab.py $p 60)"; sleep 5; done 2>&1 | tee -a gpurun_out/lab53.txt
echo "if5 $(bash tools/lab/with_lib.sh if5 python tools/lab/power_lab.py alt 60)" | tee -a gpurun_out/lab53.txt
