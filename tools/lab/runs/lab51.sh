# MrgSN in the Leap Frog transposed fill (lsn vs lif) and the stream-per-lane / f64 fills (vsn, vif vs FF default lsn)
mkdir -p gpurun_out
B=tools/lab/build
for r in 1 2; do for v in lif lsn; do
  echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py mrg 6 | tail -1)"
done; done 2>&1 | tee gpurun_out/lab51.txt
for v in lsn vsn vif; do echo "$v $(timeout 200 $B/fill_lab $B/libshv_$v.so 10)"; done 2>&1 | tee -a gpurun_out/lab51.txt
