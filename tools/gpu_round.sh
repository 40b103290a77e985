#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of the fills.
# usage (under gpurun): bash tools/gpu_round.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parts > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mrg_fill_tma|philox_fill_fast" -s 2 -c 2 \
  -o gpurun_out/prof_fill_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parts > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mrg_mc|philox_mc" -s 2 -c 2 \
  -o gpurun_out/prof_mc_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_mc_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mtgp_kernel|audit_insert|audit_second" -c 3 \
  -o gpurun_out/prof_next_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_next_$TAG.log 2>&1
ncu -i gpurun_out/prof_next_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_full_next_details_$TAG.csv 2>/dev/null
ls gpurun_out
python tools/ncu_summary.py gpurun_out/ncu_traffic_$TAG.json mrg=gpurun_out/prof_fill_$TAG.ncu-rep:mrg_fill \
  philox=gpurun_out/prof_fill_$TAG.ncu-rep:philox_fill mc_mrg=gpurun_out/prof_mc_$TAG.ncu-rep:mrg_mc \
  mc_philox=gpurun_out/prof_mc_$TAG.ncu-rep:philox_mc > /dev/null 2>&1
for r in fill mc; do ncu -i gpurun_out/prof_${r}_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_full_${r}_details_$TAG.csv 2>/dev/null; done
ls gpurun_out
