"""Lab: one fused MC pi launch at the C4 shape (2^20 streams x 2^18 samples) for ncu / timing.
   python tools/lab/mc_lab.py [mrg|philox] [reps] [samples_log2] [streams_log2] [first]
   (streams_log2 = 17, first = r * 2^17: the rank-r slice of C4 at G = 8)"""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "philox"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
samples = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 18)
ns = 1 << (int(sys.argv[4]) if len(sys.argv) > 4 else 20)
first = int(sys.argv[5]) if len(sys.argv) > 5 else 0
if which == "mrg":
    st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
    h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], first, ns, shv.SHV_SPACING_SUBSTREAM, st, 0, 0, None)
else:
    h = shv.shv_streams_create_ex(shv.SHV_GEN_PHILOX4X32_10, [12345], first, ns, 0, None, 0, 0, None)
hits = torch.zeros(1, dtype=torch.int64, device="cuda")
for r in range(reps):
    hits.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    shv.shv_mc_pi(h, samples, hits, None)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"mc {which}: {ms:.2f} ms, {ns * samples / ms / 1e6:.1f} Gsamples/s, hits {int(hits.item())}")
shv.shv_streams_destroy(h)
