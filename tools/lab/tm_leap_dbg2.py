import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1412_8266_b200 as shv, workloads as W
S = [1, *W.TINYMT32_CHECK_PARAMS]
step = sys.argv[1]
h = shv.shv_streams_create_leapfrog(W.TINYMT32, S, 70, 3, 50, None, 0, 0, None)
if step == "seg8":
    shv.shv_set_launch_config(h, 1, 64, 8)
    o = torch.empty(50 * 300, dtype=torch.int32, device="cuda"); shv.shv_generate_u32(h, o, 300, None)
elif step == "host":
    o = torch.empty(50 * 64, dtype=torch.int32, pin_memory=True); shv.shv_generate_u32_host(h, o, 64, None)
elif step == "mc":
    hits = torch.zeros(1, dtype=torch.int64, device="cuda"); c = torch.zeros(50, dtype=torch.int64, device="cuda")
    shv.shv_mc_pi_ex(h, 500, hits, c, None)
torch.cuda.synchronize()
print("ok", step, flush=True)
