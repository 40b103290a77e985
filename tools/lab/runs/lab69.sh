# transposed TinyMT32 Leap Frog: box height 128 / 64 / 32 player rows (more resident warps with smaller boxes)
mkdir -p gpurun_out
for r in 1 2; do for v in tr128 tr64 tr32; do echo "$v $(bash tools/lab/with_lib.sh $v python tools/lab/leap_lab.py tinymt 5 | awk '{print $4, $6}' | tr '\n' ' ')"; done; done 2>&1 | tee gpurun_out/lab69.txt
