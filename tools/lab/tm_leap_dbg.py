import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1412_8266_b200 as shv, workloads as W
S = [1, *W.TINYMT32_CHECK_PARAMS]
h = shv.shv_streams_create_leapfrog(W.TINYMT32, S, 70, 3, 50, None, 0, 0, None)
o = torch.empty(50 * 37, dtype=torch.int32, device="cuda"); shv.shv_generate_u32(h, o, 37, None); torch.cuda.synchronize(); print("gen37 ok", flush=True)
shv.shv_jump(h, 0, 1001)
o = torch.empty(50 * 300, dtype=torch.int32, device="cuda"); shv.shv_generate_u32(h, o, 300, None); torch.cuda.synchronize(); print("gen300 ok", flush=True)
shv.shv_set_launch_config(h, 1, 64, 8)
o = torch.empty(50 * 300, dtype=torch.int32, device="cuda"); shv.shv_generate_u32(h, o, 300, None); torch.cuda.synchronize(); print("gen300 seg8 ok", flush=True)
