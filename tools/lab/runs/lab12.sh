B=tools/lab/build
timeout 300 ncu --set full --import-source on --clock-control none -k regex:mrg_fill_rows -s 2 -c 1 -o gpurun_out/lab12_r3if5 $B/fill_lab $B/libshv_r3if5.so 1 256 0 1 > gpurun_out/lab12_ncu.log 2>&1
tail -2 gpurun_out/lab12_ncu.log
