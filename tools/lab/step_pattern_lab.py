"""Lab: why is the MRG fill slower inside the bench step (3.77 ms) than alone (3.47)?
Times the C5 MRG fill under different step patterns, with NVML clocks/power."""
import sys
import os
import time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402
import pynvml  # noqa: E402

pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)
ns, n = 1 << 20, 4096
st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
out = torch.empty(ns * n, dtype=torch.int32, device="cuda")


def fill(gen, ev=None):
    if gen == "mrg":
        h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, 1, st, 0, 0, None)
    else:
        h = shv.shv_streams_create_ex(shv.SHV_GEN_PHILOX4X32_10, [12345], 0, ns, 0, None, 0, 0, None)
    if ev:
        ev[0].record()
    shv.shv_generate_u32(h, out, n, None)
    if ev:
        ev[1].record()
    shv.shv_streams_destroy(h)


def run(name, pattern, reps=30, sleep=0.0):
    ts = {"mrg": [], "philox": []}
    clk, pw = [], []
    for r in range(reps):
        for g in pattern:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            fill(g, ev)
            torch.cuda.synchronize()
            ts[g].append(ev[0].elapsed_time(ev[1]))
        clk.append(pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM))
        pw.append(pynvml.nvmlDeviceGetPowerUsage(hd) / 1000)
        if sleep:
            time.sleep(sleep)
    med = {k: sorted(v)[len(v) // 2] for k, v in ts.items() if v}
    print(f"{name:28s} " + " ".join(f"{k} {v:.3f} ms" for k, v in med.items()) +
          f"  sm_clk {sorted(clk)[len(clk)//2]} MHz (min {min(clk)})  power {sorted(pw)[len(pw)//2]:.0f} W")


for g in ("mrg", "philox"):
    fill(g)
torch.cuda.synchronize()
run("mrg only", ["mrg"])
run("philox only", ["philox"])
run("alternate", ["mrg", "philox"])
run("alternate, 50 ms rest", ["mrg", "philox"], sleep=0.05)
run("mrg only, 50 ms rest", ["mrg"], sleep=0.05)
run("mrg only again", ["mrg"])
