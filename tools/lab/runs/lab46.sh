timeout 1200 python -m pytest tests/test_gpu_rows.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/lab46.txt
sleep 20
python tools/lab/sweep_lab.py 2>&1 | tee -a gpurun_out/lab46.txt
