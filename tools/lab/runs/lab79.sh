# TinyMT32: right shifts by constants as IMAD.HI (th1) vs SHF (th0): plain fill and transposed Leap Frog
mkdir -p gpurun_out
for r in 1 2; do for v in th0 th1; do echo "$v plain $(bash tools/lab/with_lib.sh $v python tools/lab/tinymt_lab.py 2>&1 | tail -1) leap $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py tinymt 4 | tail -1 | awk '{print $4}')"; done; done 2>&1 | tee gpurun_out/lab79.txt
