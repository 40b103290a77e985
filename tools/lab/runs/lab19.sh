# Leap Frog transposed fills at the C5 shape: timings and ncu --set full
mkdir -p gpurun_out
for g in philox mrg; do python tools/lab/leap_lab.py $g 3; done 2>&1 | tee gpurun_out/lab19_leap.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"leap_ctr_tr|leap_mrg_tr" -c 1 -o gpurun_out/lab19_leap_philox python tools/lab/leap_lab.py philox 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"leap_ctr_tr|leap_mrg_tr" -c 1 -o gpurun_out/lab19_leap_mrg python tools/lab/leap_lab.py mrg 1 > /dev/null 2>&1
ls gpurun_out | grep lab19
python - <<'PY' 2>&1 | tee -a gpurun_out/lab19_leap.txt
import torch, sys
sys.path.insert(0, '.')
import paper_1412_8266_b200 as shv
ns, n = 1 << 20, 4096
out = torch.empty(ns * n, dtype=torch.int32, device='cuda')
h = shv.shv_streams_create_ex(shv.SHV_GEN_THREEFRY4X64_20, [12345], 0, ns, 0, None, 0, 0, None)
for r in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); shv.shv_generate_u32(h, out, n, None); b.record(); torch.cuda.synchronize()
    print('threefry fill', round(a.elapsed_time(b), 3), 'ms')
PY
timeout 600 python -m pytest tests -m gpu -q -k "threefry or Threefry" 2>&1 | tail -2 | tee -a gpurun_out/lab19_leap.txt
