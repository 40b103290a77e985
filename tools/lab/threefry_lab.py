"""Lab: Threefry4x64-20 u32 fill at the C5 shape (2^20 counter-streams x 4096)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402

ns, n = 1 << 20, 4096
h = shv.shv_streams_create_ex(shv.SHV_GEN_THREEFRY4X64_20, [12345], 0, ns, 0, None, 0, 0, None)
out = torch.empty(ns * n, dtype=torch.int32, device="cuda")
for r in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    shv.shv_generate_u32(h, out, n, None)
    b.record()
    torch.cuda.synchronize()
    print(f"threefry fill: {a.elapsed_time(b):.3f} ms  checksum {int(out.view(torch.int64).sum().item()) & ((1 << 64) - 1):016x}")
shv.shv_streams_destroy(h)
