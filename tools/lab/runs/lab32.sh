timeout 900 python -m pytest tests/test_gpu_rows.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/lab32.txt
python - <<'PY' 2>&1 | tee -a gpurun_out/lab32.txt
import torch, sys
sys.path.insert(0, '.')
import paper_1412_8266_b200 as shv
out = torch.empty(1 << 32, dtype=torch.int32, device='cuda')
for lg in (13, 14, 15, 16, 17, 18, 19, 20, 21, 22):
    ns = 1 << lg; n = (1 << 32) // ns
    st = torch.empty(6 * ns, dtype=torch.int32, device='cuda')
    ts = []
    for r in range(4):
        h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, 1, st, 0, 0, None)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); shv.shv_generate_u32(h, out, n, None); b.record(); torch.cuda.synchronize()
        shv.shv_streams_destroy(h)
        if r: ts.append(a.elapsed_time(b))
    ms = sorted(ts)[1]
    print(f"2^{lg} streams x {n}: {ms:.3f} ms  {(1<<32)/ms/1e6:.1f} Gnumbers/s")
PY
