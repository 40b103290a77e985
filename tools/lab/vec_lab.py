"""Lab: MRG32k3a fills that do not split into row tiles (stream-per-lane TMA u32, staged f64 vector
path, scalar path): 2^20 streams x 4104 u32 (n % 128 != 0), 2^19 x 4104 f64, 2^20 x 4101 u32 (scalar)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402

for ns, n, kind in ((1 << 20, 4104, "u32"), (1 << 19, 4104, "f64"), (1 << 18, 4101, "u32")):
    st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
    h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, shv.SHV_SPACING_SUBSTREAM, st, 0, 0, None)
    out = torch.empty(ns * n, dtype=torch.int32 if kind == "u32" else torch.float64, device="cuda")
    fn = shv.shv_generate_u32 if kind == "u32" else shv.shv_generate_f64
    ts = []
    for r in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(h, out, n, None)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ck = int(out.view(torch.int64).sum().item()) & ((1 << 64) - 1)
    print(f"{ns}x{n} {kind}: best {min(ts[1:]):.3f} ms  checksum {ck:016x}")
    shv.shv_streams_destroy(h)
