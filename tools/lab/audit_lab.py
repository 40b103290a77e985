"""Lab: disjointness audit of 2^18 x 4096 MRG32k3a C3 rows (1.07e9 windows).
   python tools/lab/audit_lab.py [reps] [log2_streams]"""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ns, n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 18), 4096
st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, shv.SHV_SPACING_SUBSTREAM, st, 0, 0, None)
rows = torch.empty(ns * n, dtype=torch.int32, device="cuda")
shv.shv_generate_u32(h, rows, n, None)
shv.shv_streams_destroy(h)
wsb = shv.shv_verify_disjoint_workspace_bytes(ns, n)
ws = torch.empty(wsb // 8, dtype=torch.int64, device="cuda")
rep = torch.zeros(7, dtype=torch.int64, device="cuda")
for r in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    shv.shv_verify_disjoint(rows, ns, n, ws, wsb, rep, None)
    b.record()
    torch.cuda.synchronize()
    print(f"audit {ns}x{n}: {a.elapsed_time(b):.2f} ms, report {rep.cpu().tolist()[:3]}")
