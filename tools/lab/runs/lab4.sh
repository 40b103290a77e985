mkdir -p gpurun_out
B=tools/lab/build
$B/step2_lab > gpurun_out/lab4_step2.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:mrg_fill_rows -s 2 -c 1 -o gpurun_out/lab4_rif4 $B/fill_lab $B/libshv_rif4.so 1 > gpurun_out/lab4_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:mrg_fill_rows -s 2 -c 1 -o gpurun_out/lab4_rff4 $B/fill_lab $B/libshv_rff4.so 1 >> gpurun_out/lab4_ncu.log 2>&1
cat gpurun_out/lab4_step2.txt; tail -3 gpurun_out/lab4_ncu.log
