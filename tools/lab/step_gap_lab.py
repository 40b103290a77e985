"""Lab: the bench step back to back (no host syncs), events around every launch, to split the
step time into kernel time and inter-kernel gaps (host latency vs power).
   python tools/lab/step_gap_lab.py [steps]"""
import os
import sys
import time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1412_8266_b200 as shv  # noqa: E402
import workloads as W  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
wm, wp = W.C5_MRG, W.C5_PHILOX
ns, n = wm.n_streams, wm.n
out = torch.empty(ns * n, dtype=torch.int32, device="cuda")
state = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
sp = torch.cuda.current_stream()


def step(ev=None):
    h = shv.shv_streams_create_ex(wm.gen, list(wm.seed), wm.first, ns, wm.spacing, state, 0, 0, sp)
    if ev: ev[0].record(sp)
    shv.shv_generate_u32(h, out, n, sp)
    if ev: ev[1].record(sp)
    shv.shv_streams_destroy(h)
    h = shv.shv_streams_create_ex(wp.gen, list(wp.seed), wp.first, ns, wp.spacing, None, 0, 0, sp)
    if ev: ev[2].record(sp)
    shv.shv_generate_u32(h, out, n, sp)
    if ev: ev[3].record(sp)
    shv.shv_streams_destroy(h)


for _ in range(3):
    step()
torch.cuda.synchronize()
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
t_host = time.perf_counter()
for i in range(steps):
    step(evs[i])
t_host = (time.perf_counter() - t_host) * 1e3
torch.cuda.synchronize()
mrg = [e[0].elapsed_time(e[1]) for e in evs]
gap1 = [e[1].elapsed_time(e[2]) for e in evs]   # MRG end -> Philox start (destroy + create + host build)
phx = [e[2].elapsed_time(e[3]) for e in evs]
gap2 = [evs[i][3].elapsed_time(evs[i + 1][0]) for i in range(steps - 1)]  # Philox end -> next MRG start (incl. seed kernel)
tot = evs[0][0].elapsed_time(evs[-1][3])
m = lambda v: round(sum(v) / len(v), 4)
print({"steps": steps, "mrg": m(mrg), "philox": m(phx), "gap_mrg_to_philox": m(gap1), "gap_philox_to_mrg": m(gap2),
       "span_ms_per_step": round(tot / steps, 4), "host_ms_per_step": round(t_host / steps, 4)})
