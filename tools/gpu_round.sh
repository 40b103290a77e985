#!/bin/bash
# One GPU session: smoke, tests, bench, ncu launch list and --set full captures
# of the fills (C5) and of the fused MC kernels (2^16 streams x 2^18 samples:
# short enough for ncu's replays), summarised into gpurun_out/ncu_traffic_TAG.json.
# usage (under gpurun): bash tools/gpu_round.sh TAG [skip-tests]
TAG=${1:-r02}
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
if [ "$2" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 600 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parts > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mrg_fill_rows|philox_fill_fast" -s 2 -c 2 \
  -o gpurun_out/prof_fill_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parts > gpurun_out/ncu_full_$TAG.log 2>&1
for g in mrg philox; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${g}_mc" -c 1 \
    -o gpurun_out/prof_mc_${g}_$TAG python tools/lab/mc_lab.py $g 1 18 16 > gpurun_out/ncu_mc_${g}_$TAG.log 2>&1
done
python tools/ncu_summary.py gpurun_out/ncu_traffic_$TAG.json mrg=gpurun_out/prof_fill_$TAG.ncu-rep:mrg_fill_rows:4294967296 \
  philox=gpurun_out/prof_fill_$TAG.ncu-rep:philox_fill:4294967296 \
  mc_mrg=gpurun_out/prof_mc_mrg_$TAG.ncu-rep:mrg_mc:17179869184 \
  mc_philox=gpurun_out/prof_mc_philox_$TAG.ncu-rep:philox_mc:17179869184 > /dev/null 2>&1
ncu -i gpurun_out/prof_fill_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_full_fill_details_$TAG.csv 2>/dev/null
for g in mrg philox; do
  ncu -i gpurun_out/prof_mc_${g}_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_full_mc_${g}_details_$TAG.csv 2>/dev/null
done
ls gpurun_out | grep $TAG
