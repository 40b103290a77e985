"""Lab: MRG32k3a u32 fill over the C6 stream-count sweep (2^32 numbers per shape), shapes
interleaved, cold (2nd launch) and back to back (mean of 6).  python tools/lab/sweep_lab.py"""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402

out = torch.empty(1 << 32, dtype=torch.int32, device='cuda')
for lg in (13, 15, 17, 19, 20, 21, 22):
    ns = 1 << lg
    n = (1 << 32) // ns
    st = torch.empty(6 * ns, dtype=torch.int32, device='cuda')
    h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, 1, st, 0, 0, None)
    ts = []
    for r in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        shv.shv_generate_u32(h, out, n, None)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    shv.shv_streams_destroy(h)
    print(f"2^{lg} x {n}: cold {ts[1]:.3f} ms, back to back mean {sum(ts[2:]) / 6:.3f} ms")
