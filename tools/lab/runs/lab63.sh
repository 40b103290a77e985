# Threefry plain fill chunk loop unrolled 1/2/4; TinyMT32 transposed Leap Frog box loop unrolled 1/2/4
mkdir -p gpurun_out
for r in 1 2; do
for v in u1 tf2 tf4; do echo "$v threefry $(bash tools/lab/with_lib.sh $v python tools/lab/threefry_lab.py | awk '{print $3}' | tr '\n' ' ')"; done
for v in u1 tm2 tm4; do echo "$v tinymt-leap $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py tinymt 5 | awk '{print $4}' | tr '\n' ' ')"; done
done 2>&1 | tee gpurun_out/lab63.txt
