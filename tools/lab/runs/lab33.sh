python - <<'PY' 2>&1 | tee gpurun_out/lab33.txt
import torch, sys
sys.path.insert(0, '.')
import paper_1412_8266_b200 as shv
out = torch.empty(1 << 32, dtype=torch.int32, device='cuda')
def t(lg, reps=6):
    ns = 1 << lg; n = (1 << 32) // ns
    st = torch.empty(6 * ns, dtype=torch.int32, device='cuda')
    h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, 1, st, 0, 0, None)
    ts = []
    for r in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); shv.shv_generate_u32(h, out, n, None); b.record(); torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 3))
    shv.shv_streams_destroy(h)
    return ts
for rnd in range(3):
    for lg in (20, 17, 21, 19, 22):
        print(rnd, f"2^{lg}", t(lg))
PY
