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


def run_b2b(name, pattern, reps=30):
    """Back to back as bench.py times the step: no host sync between fills, NVML sampled every 2 ms."""
    import threading
    hs = {"mrg": shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, 1, st, 0, 0, None),
          "philox": shv.shv_streams_create_ex(shv.SHV_GEN_PHILOX4X32_10, [12345], 0, ns, 0, None, 0, 0, None)}
    evs = []
    samples, stop = [], [False]

    def sampler():
        while not stop[0]:
            samples.append((pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(hd) / 1000))
            time.sleep(0.002)
    th = threading.Thread(target=sampler)
    th.start()
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
    ts = {"mrg": [], "philox": []}
    for g, ev in evs:
        ts[g].append(ev[0].elapsed_time(ev[1]))
    med = {k: sorted(v)[len(v) // 2] for k, v in ts.items() if v}
    clk = sorted(c for c, _ in samples)
    pw = sorted(p for _, p in samples)
    print(f"{name:28s} " + " ".join(f"{k} {v:.3f} ms" for k, v in med.items()) +
          f"  sm_clk median {clk[len(clk)//2]} min {clk[0]} MHz  power median {pw[len(pw)//2]:.0f} max {pw[-1]:.0f} W  ({len(samples)} samples)")
    for h in hs.values():
        shv.shv_streams_destroy(h)


run_b2b("b2b mrg only", ["mrg"], reps=60)
run_b2b("b2b philox only", ["philox"], reps=60)
run_b2b("b2b alternate", ["mrg", "philox"], reps=40)
run_b2b("b2b mrg only again", ["mrg"], reps=60)
