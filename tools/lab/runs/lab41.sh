for r in 1 2; do for v in tr256 tr128; do
  echo "$v plain $(bash tools/lab/with_lib.sh $v python tools/lab/tinymt_lab.py 2>&1 | tail -1)"
done; done 2>&1 | tee gpurun_out/lab41.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "tinymt or TinyMT" 2>&1 | tail -2 | tee -a gpurun_out/lab41.txt
