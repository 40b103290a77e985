# power limits of the box and NVML power/clock reasons during a sustained MRG fill
mkdir -p gpurun_out
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE > gpurun_out/lab57_smi.txt 2>&1
python - <<'PY' > gpurun_out/lab57_run.txt 2>&1 &
import subprocess, sys
subprocess.run([sys.executable, "tools/lab/power_lab.py", "mrg", "400"])
PY
PID=$!
sleep 3
for i in 1 2 3 4 5 6; do nvidia-smi --query-gpu=power.draw,power.draw.instant,power.limit,enforced.power.limit,clocks.sm,clocks_throttle_reasons.active,temperature.gpu --format=csv,noheader >> gpurun_out/lab57_q.txt 2>&1; sleep 0.2; done
wait $PID
cat gpurun_out/lab57_q.txt gpurun_out/lab57_run.txt; grep -i -A3 "Power Limit\|Power Draw\|Throttle\|Clocks Event" gpurun_out/lab57_smi.txt | head -60
