"""Lab: sustained (back-to-back) C5 fills with NVML clocks and power sampled every 2 ms.
   python tools/lab/power_lab.py [mrg|philox|alt] [reps]   (run under tools/lab/with_lib.sh for lab builds)"""
import os
import sys
import threading
import time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402
import pynvml  # noqa: E402

pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)
which = sys.argv[1] if len(sys.argv) > 1 else "mrg"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
ns, n = 1 << 20, 4096
st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
out = torch.empty(ns * n, dtype=torch.int32, device="cuda")
hs = {"mrg": shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, 1, st, 0, 0, None),
      "philox": shv.shv_streams_create_ex(shv.SHV_GEN_PHILOX4X32_10, [12345], 0, ns, 0, None, 0, 0, None)}
pattern = ["mrg", "philox"] if which == "alt" else [which]
for g in pattern:  # warm-up
    shv.shv_generate_u32(hs[g], out, n, None)
torch.cuda.synchronize()
samples, stop = [], [False]


def sampler():
    while not stop[0]:
        samples.append((pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(hd) / 1000))
        time.sleep(0.002)


th = threading.Thread(target=sampler)
th.start()
evs = []
for r in range(reps):
    for g in pattern:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
        shv.shv_generate_u32(hs[g], out, n, None)
        ev[1].record()
        evs.append((g, ev))
torch.cuda.synchronize()
stop[0] = True
th.join()
ts = {g: [] for g in pattern}
for g, ev in evs:
    ts[g].append(ev[0].elapsed_time(ev[1]))
clk = sorted(c for c, _ in samples)
pw = sorted(p for _, p in samples)
res = {g: {"mean": round(sum(v) / len(v), 4), "median": round(sorted(v)[len(v) // 2], 4), "best": round(min(v), 4),
           "last10": round(sum(v[-10:]) / 10, 4)} for g, v in ts.items()}
print({"pattern": which, **res, "sm_clk_median": clk[len(clk) // 2], "sm_clk_min": clk[0],
       "power_median": round(pw[len(pw) // 2]), "power_max": round(pw[-1]), "samples": len(samples)})
