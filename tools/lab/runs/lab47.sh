mkdir -p gpurun_out
timeout 120 tools/lab/build/step4_lab > gpurun_out/lab47_step4.txt 2>&1
cat gpurun_out/lab47_step4.txt
