import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1412_8266_b200 as shv, oracle as orc, workloads as W
for K, first, n, m in ((1000, 16, 300, 1024), (1000, 17, 300, 1024), (1000, 17, 300, 64), (1000, 0, 128, 32), (8, 0, 8, 64)):
    h = shv.shv_streams_create_leapfrog(W.PHILOX4X32_10, [12345, 678], K, first, n, None, 0, 0, None)
    out = torch.empty(n * m, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, out, m, None); torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32).reshape(n, m)
    want = orc.generate(W.PHILOX4X32_10, [12345, 678], n, m, first=first, spacing=W.SPACING_LEAPFROG, players=K)
    bad = np.nonzero((got != want).any(axis=1))[0]
    cols = np.nonzero((got != want).any(axis=0))[0]
    print(K, first, n, m, "bad rows", len(bad), bad[:12], "bad cols", len(cols), cols[:8])
    shv.shv_streams_destroy(h)
