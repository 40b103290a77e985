"""Lab: TinyMT32 u32 fill at the C5 shape (2^20 streams x 4096, groups of 256)."""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402
import workloads as W  # noqa: E402

ns, n = 1 << 20, 4096
params = W.tinymt32_test_params(ns // 256 + 1)
st = torch.empty(4 * ns, dtype=torch.int32, device="cuda")
h = shv.shv_streams_create_tinymt32(params, 12345, 256, 0, ns, st, 0, 0, None)
out = torch.empty(ns * n, dtype=torch.int32, device="cuda")
for r in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    shv.shv_generate_u32(h, out, n, None)
    b.record()
    torch.cuda.synchronize()
    print(f"tinymt fill: {a.elapsed_time(b):.3f} ms")
shv.shv_streams_destroy(h)
