python - <<'PY' 2>&1 | tee gpurun_out/lab36.txt
import torch, sys, time, threading
sys.path.insert(0, '.')
import paper_1412_8266_b200 as shv
import pynvml
pynvml.nvmlInit(); hd = pynvml.nvmlDeviceGetHandleByIndex(0)
ns = 1 << 20
st = torch.empty(6 * ns, dtype=torch.int32, device='cuda')
hits = torch.zeros(1, dtype=torch.int64, device='cuda')
for gen in ('mrg', 'philox'):
    for it in range(2):
        if gen == 'mrg':
            h = shv.shv_streams_create_ex(shv.SHV_GEN_MRG32K3A, [12345], 0, ns, 1, st, 0, 0, None)
        else:
            h = shv.shv_streams_create_ex(shv.SHV_GEN_PHILOX4X32_10, [12345], 0, ns, 0, None, 0, 0, None)
        samples, stop = [], [False]
        def sampler():
            while not stop[0]:
                samples.append((pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(hd) / 1000,
                                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hd)))
                time.sleep(0.005)
        th = threading.Thread(target=sampler); th.start()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); shv.shv_mc_pi(h, 1 << 18, hits, None); b.record(); torch.cuda.synchronize()
        stop[0] = True; th.join()
        shv.shv_streams_destroy(h)
        clk = [c for c, _, _ in samples]; pw = [p for _, p, _ in samples]
        reasons = set(r for _, _, r in samples)
        print(gen, it, round(a.elapsed_time(b), 1), 'ms; sm clk min/median/max', min(clk), sorted(clk)[len(clk)//2], max(clk),
              'power median/max', round(sorted(pw)[len(pw)//2]), round(max(pw)), 'throttle masks', sorted(hex(x) for x in reasons))
        time.sleep(2)
PY
