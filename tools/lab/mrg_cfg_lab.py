"""Lab: C5 MRG32k3a u32 fill (2^20 substreams x 4096) under launch configurations
(blocks per SM, threads per block, segment length) — results never change (R10)."""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402

ns, n = 1 << 20, 4096
st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
out = torch.empty(ns * n, dtype=torch.int32, device="cuda")
ref = None
for bps, tpb, seg in ((0, 0, 0), (0, 128, 0), (0, 64, 0), (2, 256, 0), (3, 256, 0), (0, 0, 1024), (0, 0, 512),
                      (0, 0, 2048), (0, 0, 4096), (0, 128, 1024)):
    h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, shv.SHV_SPACING_SUBSTREAM, st, 0, 0, None)
    shv.shv_set_launch_config(h, bps, tpb, seg)
    ts = []
    for r in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        shv.shv_generate_u32(h, out, n, None)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    cs = int(out[::9973].sum().item())
    ref = cs if ref is None else ref
    print(f"bps {bps} tpb {tpb} seg {seg}: {min(ts[1:]):.3f} ms  {'ok' if cs == ref else 'MISMATCH'}")
    shv.shv_streams_destroy(h)
