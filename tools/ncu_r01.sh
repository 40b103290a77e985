set -x
./tools/pipe_microbench > gpurun_out/microbench.json 2>&1
cat gpurun_out/microbench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parts > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mrg_fill|philox_fill_fast" -s 2 -c 2 -o gpurun_out/prof_fill_r01 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parts > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
