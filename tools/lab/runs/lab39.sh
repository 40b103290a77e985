for r in 1 2; do for v in tm0 tm1; do
  echo "$v plain $(bash tools/lab/with_lib.sh $v python tools/lab/tinymt_lab.py 2>&1 | tail -1)"
  echo "$v leap $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py tinymt 4 | tail -1)"
done; done 2>&1 | tee gpurun_out/lab39.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "tinymt or TinyMT or device_api or leap" 2>&1 | tail -2 | tee -a gpurun_out/lab39.txt
