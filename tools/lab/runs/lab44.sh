timeout 1200 python -m pytest tests/test_gpu_rows.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/lab44.txt
sed -n 1,200p tools/lab/runs/lab32.sh | sed -n '/python - <<.PY./,/^PY$/p' > /tmp/sweep.sh
bash /tmp/sweep.sh 2>&1 | tee -a gpurun_out/lab44.txt
