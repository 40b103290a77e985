"""Lab: one Leap Frog fill at the C5 shape (2^20 players x 4096 u32) for ncu.
   python tools/lab/leap_lab.py [mrg|philox|threefry|tinymt] [reps]"""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "philox"
gen = {"mrg": shv.SHV_GEN_MRG32K3A, "philox": shv.SHV_GEN_PHILOX4X32_10, "threefry": shv.SHV_GEN_THREEFRY4X64_20,
       "tinymt": shv.SHV_GEN_TINYMT32}[which]
seed = {"tinymt": [12345, 0x8F7011EE, 0xFC78FF1F, 0x3793FDFF]}.get(which, [12345])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
K, n = 1 << 20, 4096
st = torch.empty(6 * K, dtype=torch.int32, device="cuda") if gen == shv.SHV_GEN_MRG32K3A else None
h = shv.shv_streams_create_leapfrog(gen, seed, K, 0, K, st, 0, 0, None)
out = torch.empty(K * n, dtype=torch.int32, device="cuda")
for r in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    shv.shv_generate_u32(h, out, n, None)
    b.record()
    torch.cuda.synchronize()
    print(f"leap fill {sys.argv[1:2]}: {a.elapsed_time(b):.3f} ms  "
          f"checksum {int(out.view(torch.int64).sum().item()) & ((1 << 64) - 1):016x}")
shv.shv_streams_destroy(h)
