#!/usr/bin/env python
"""Benchmark of the ShoveRand hot path on B200 (arXiv 1412.8266).

Workload (BASELINE.json configs[4], "C5"; the metric is quoted on it): every
rank fills 16 GiB = 2^20 streams x 4096 u32 from MRG32k3a (substreams of seed
12345) and 16 GiB from Philox4x32-10 (counter-streams, key 12345); rank r owns
streams [r*2^20, (r+1)*2^20) (weak scaling, no collective on the data path).
One step = the whole bulk path for both generators: create (seed validation,
jump-table products, per-stream start states) -> generate_u32 -> destroy.
value = u32 numbers produced by all ranks / max-over-ranks device time.

Also reported (same JSON line): per-kernel timings and the HBM-write roofline
of the dominant kernel, the fused Monte Carlo pi (configs[3], strong scaling,
one NCCL all_reduce of the hit count), the f64 fill (configs[2]), the oracle
CPU baseline, e2e through shv_generate_u32_host (pinned host buffer), clocks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl shv|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import random
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "Gnumbers/s (u32) per GPU and box at 1/2/4/8 B200; % of HBM-write roofline"
UNIT = "Gnumbers/s"
WORKLOAD = ("C5: bulk fill 16 GiB u32 per GPU from MRG32k3a (2^20 substreams x 4096, seed 12345) "
            "and Philox4x32-10 (2^20 counter-streams x 4096, key 12345); rank r owns streams "
            "[r*2^20,(r+1)*2^20)")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(kernel_key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        v = d.get(kernel_key)
        if v:
            return float(v["dram_bytes_read"] + v["dram_bytes_write"])
    return None


def profile_record(kernel_key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(kernel_key)


# Issue roofline of the compute-bound kernels ("for the compute-bound
# MC pi, the percentage is of the integer-pipe / issue roofline"): 148 SMs x 4
# schedulers x 1 warp instruction per clock at the 1965 MHz maximum SM clock
# (B200_PROFILING.md) = 1.163 T warp instructions/s.
ISSUE_PEAK = 148 * 4 * 1.965e9


def limiter_from_profiles(kernel_key):
    """What ncu says binds the kernel (profiles/ncu_traffic.json), for the reader."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    v = json.load(open(p)).get(kernel_key)
    if not v:
        return None
    pipes = {"fp64": v.get("fp64_pipe_pct"), "fma_heavy": v.get("fmaheavy_pipe_pct"),
             "alu": v.get("alu_pipe_pct"), "issue": v.get("issue_active_pct")}
    pipes = {k: x for k, x in pipes.items() if isinstance(x, (int, float)) and x == x}
    if not pipes:
        return None
    top = max(pipes, key=lambda k: pipes[k])
    return f"ncu: {top} {pipes[top]:.0f}% busy ({', '.join(f'{k} {x:.0f}%' for k, x in pipes.items() if x is not None)})"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpus):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,clocks.mem,power.draw")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-i", ",".join(str(g) for g in gpus), "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.count(",") >= 7]
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].strip().isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].strip().isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k].strip() == "Active"})
        busy = [s for s in sm if s > 0.5 * mx] or sm
        out = {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}

        def med(col):
            v = []
            for r in rows:
                try:
                    v.append(float(r[col]))
                except (IndexError, ValueError):
                    pass
            return statistics.median(v) if v else None
        out["mem_mhz"], out["power_w"] = med(8), med(9)
        return out


# ---------------------------------------------------------------------------- oracle arm

def _oracle_run(k: int, threads: int) -> float:
    """Oracle (as it stands) on the first k streams x 4096 u32 of each C5
    generator; returns seconds."""
    import oracle
    n = W.C5_MRG.n
    t = time.perf_counter()
    for s0 in range(0, k, 1 << 14):  # 256 MiB chunks: bounded host memory
        ns = min(1 << 14, k - s0)
        oracle.generate(W.MRG32K3A, list(W.C5_MRG.seed), ns, n, first=s0, spacing=W.C5_MRG.spacing,
                        nthreads=threads)
        oracle.generate(W.PHILOX4X32_10, list(W.C5_PHILOX.seed), ns, n, first=s0,
                        spacing=W.C5_PHILOX.spacing, nthreads=threads)
    return time.perf_counter() - t


def _oracle_calibrate(target_s: float, threads: int) -> int:
    """Stream-prefix length k whose oracle run takes about target_s seconds."""
    k = max(threads, 16)
    while True:
        t = _oracle_run(k, threads)
        if t >= 1.0 or k >= W.C5_MRG.n_streams:
            break
        k = min(W.C5_MRG.n_streams, k * 4)
    return max(1, min(W.C5_MRG.n_streams, int(k * target_s / max(t, 1e-3))))


def _sample_desc(k: int, threads: int) -> str:
    return (f"first {k} of 2^20 streams x {W.C5_MRG.n} u32 from each of MRG32k3a and "
            f"Philox4x32-10 (C5 prefix), {threads} threads")


def cpu_baseline(threads):
    k = _oracle_calibrate(12.0, threads)
    t = _oracle_run(k, threads)
    # the oracle single-threaded as well as on all host threads
    k1 = _oracle_calibrate(3.0, 1)
    t1 = _oracle_run(k1, 1)
    return {"value": 2 * k * W.C5_MRG.n / t / 1e9, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": _sample_desc(k, threads), "seconds": round(t, 3),
            "single_thread": {"value": 2 * k1 * W.C5_MRG.n / t1 / 1e9, "unit": UNIT, "cores": 1,
                              "sample": _sample_desc(k1, 1), "seconds": round(t1, 3)}}


def _oracle_mc(k: int, threads: int) -> tuple:
    """Oracle dartboard counts (C4 shape: 2^18 samples per stream) on the first
    k streams of each generator; returns (seconds, samples)."""
    import oracle
    t = time.perf_counter()
    for w in (W.C4_MRG, W.C4_PHILOX):
        oracle.mc_count(w.gen, list(w.seed), k, w.n, spacing=w.spacing, nthreads=threads)
    return time.perf_counter() - t, 2 * k * W.C4_MRG.n


def cpu_baseline_mc(threads):
    """the oracle on a C4 subset (1024 streams), on all host threads
    and single-threaded (on 32 streams)."""
    t, ns = _oracle_mc(1024, threads)
    t1, ns1 = _oracle_mc(32, 1)
    desc = "first {k} of 2^20 streams x 2^18 samples, MRG32k3a and Philox4x32-10 (C4 subset), {t} threads"
    return {"value": ns / t / 1e9, "unit": "Gsamples/s", "cores": threads, "kind": "oracle",
            "sample": desc.format(k=1024, t=threads), "seconds": round(t, 3),
            "single_thread": {"value": ns1 / t1 / 1e9, "unit": "Gsamples/s", "cores": 1,
                              "sample": desc.format(k=32, t=1), "seconds": round(t1, 3)}}


def run_reference(args, rank, world):
    """--impl reference: the oracle, as it stands, on the host cores; rank 0 only."""
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    import oracle
    oracle.build()
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    k = _oracle_calibrate(per_step, threads)
    for w in range(args.warmup):
        t = _oracle_run(k, threads)
        if w == 0 and abs(t / per_step - 1.0) > 0.2:  # the short calibration runs mis-scale: re-aim once
            k = max(1, min(W.C5_MRG.n_streams, int(k * per_step / max(t, 1e-3))))
    tot_t = 0.0
    for _ in range(args.steps):
        tot_t += _oracle_run(k, threads)
    value = 2 * k * W.C5_MRG.n * args.steps / tot_t / 1e9
    desc = _sample_desc(k, threads)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / max(1, args.steps), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "sample": desc},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="shv", choices=["shv", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parts", action="store_true")
    ap.add_argument("--small", action="store_true",
                    help="test mode: 2^14 streams per rank, 2^12 MC samples per stream (not a bench number)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: validate the N>1 logic with ranks sharing a GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "shv" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # under torchrun the process group (and the Monte Carlo all_reduce) is set
    # up even at world size 1, so the NCCL path runs on a one-GPU box too;
    # NCCL's init log (nranks, transports, NVLS) stays on stderr
    launched = "TORCHELASTIC_RUN_ID" in os.environ or world > 1
    if launched and args.backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_1412_8266_b200 as shv

    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if launched:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    def shrink(w, mc=False):
        if not args.small:
            return w
        return W.Workload(w.name + "-small", w.gen, w.seed, min(w.n_streams, 1 << 14),
                          min(w.n, 1 << 12) if mc else w.n, w.spacing, w.first)

    wm = W.rank_slice(shrink(W.C5_MRG), rank, world, weak=True)
    wp = W.rank_slice(shrink(W.C5_PHILOX), rank, world, weak=True)
    n = wm.n
    total_per_rank = wm.n_streams * n  # per generator
    out = torch.empty(total_per_rank, dtype=torch.int32, device=dev)  # 16 GiB
    state = torch.empty(6 * wm.n_streams, dtype=torch.int32, device=dev)
    ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(2)] for k in ("mrg", "philox")}
    kt = {"mrg": [], "philox": []}

    def step(timed_kernels=False):
        h = shv.shv_streams_create_ex(wm.gen, list(wm.seed), wm.first, wm.n_streams, wm.spacing,
                                      state, 0, local, sp)
        if timed_kernels:
            ev["mrg"][0].record(stream)
        shv.shv_generate_u32(h, out, n, sp)
        if timed_kernels:
            ev["mrg"][1].record(stream)
        shv.shv_streams_destroy(h)
        h = shv.shv_streams_create_ex(wp.gen, list(wp.seed), wp.first, wp.n_streams, wp.spacing,
                                      None, 0, local, sp)
        if timed_kernels:
            ev["philox"][0].record(stream)
        shv.shv_generate_u32(h, out, n, sp)
        if timed_kernels:
            ev["philox"][1].record(stream)
        shv.shv_streams_destroy(h)

    for _ in range(args.warmup):
        step()
    clocks = Clocks([local] if world == 1 else list(range(min(world, torch.cuda.device_count())))) if rank == 0 else None
    time.sleep(0.3)  # let the sampler start before the measured loops
    # per-kernel durations (same launches as the step, events on the launching stream)
    for _ in range(args.steps):
        step(timed_kernels=True)
        torch.cuda.synchronize()
        for k in kt:
            kt[k].append(ev[k][0].elapsed_time(ev[k][1]))

    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    barrier()
    ms = max_over_ranks(t0.elapsed_time(t1))
    clk = clocks.stop() if clocks else None
    ms_step = ms / args.steps
    numbers = 2 * total_per_rank * world * args.steps
    value = numbers / (ms * 1e-3) / 1e9

    peak, peak_src = peaks()
    kms = {k: statistics.mean(v) for k, v in kt.items()}
    dom = max(kms, key=kms.get)
    alg_bytes = 4 * total_per_rank  # u32 written per launch (4 B/number, 0 read)
    achieved = alg_bytes / (kms[dom] * 1e-3) / 1e9
    hbm = {"bound": "hbm", "kernel": "mrg_fill_rows_kernel<u32>" if dom == "mrg" else "philox_fill_fast_kernel<u32>",
           "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "peak_source": peak_src,
           "traffic": traffic_from_profiles(dom),
           "limiter": limiter_from_profiles(dom),
           "algorithmic_bytes_per_launch": alg_bytes}
    # the metric's roofline is the HBM write of 4 B per number (0 B
    # read) for the dominant kernel. What ncu says keeps the kernel from it (the
    # step's pipe mix and issue rate, profiles/ncu_traffic.json) is in `limiter`
    # and `pipes`; the MRG32k3a step is compute-bound at ~17-19 issue slots per
    # number and, run back to back, power-limited.
    rec = profile_record(dom) or {}
    hbm["pipes"] = {k: rec.get(k) for k in ("issue_active_pct", "fp64_pipe_pct", "fmaheavy_pipe_pct",
                                              "alu_pipe_pct") if rec.get(k) is not None}
    if rec.get("inst_per_unit"):
        hbm["issue"] = {"inst_per_number": round(rec["inst_per_unit"], 3),
                        "achieved": round(rec["inst_per_unit"] * total_per_rank / (kms[dom] * 1e-3) / 1e12, 4),
                        "peak": round(ISSUE_PEAK / 1e12, 4), "unit": "T warp instr/s",
                        "frac": round(rec["inst_per_unit"] * total_per_rank / (kms[dom] * 1e-3) / ISSUE_PEAK, 4)}
    roof = hbm
    parts = {k: {"ms": round(kms[k], 4), "Gnumbers_per_s": round(total_per_rank / (kms[k] * 1e-3) / 1e9, 1),
                 "GB_per_s": round(alg_bytes / (kms[k] * 1e-3) / 1e9, 1),
                 "frac_of_hbm_peak": round(alg_bytes / (kms[k] * 1e-3) / 1e9 / peak, 4)}
             for k in kms}

    # ---- fused Monte Carlo pi (configs[3]) and f64 fill (configs[2]) ----
    if not args.no_parts:
        for w0 in (W.C4_MRG, W.C4_PHILOX):
            w = shrink(w0, mc=True)
            ws = W.rank_slice(w, rank, world, weak=False)
            st = torch.empty(6 * ws.n_streams, dtype=torch.int32, device=dev)
            hits = torch.zeros(1, dtype=torch.int64, device=dev)
            times = []
            for it in range(3):
                h = shv.shv_streams_create_ex(ws.gen, list(ws.seed), ws.first, ws.n_streams, ws.spacing,
                                              st if ws.gen == W.MRG32K3A else None, 0, local, sp)
                hits.zero_()
                barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                shv.shv_mc_pi(h, ws.n, hits, sp)
                if launched:
                    dist.all_reduce(hits)  # NCCL: one int64 per rank
                b.record(stream)
                barrier()
                shv.shv_streams_destroy(h)
                times.append(max_over_ranks(a.elapsed_time(b)))
            tot = int(hits.item())
            N = w.n_streams * w.n
            import math
            p = 221069946527026 / 2 ** 48
            pi_hat = 4 * tot / N
            t_ms = min(times)
            key = "mc_pi_" + ("mrg" if w.gen == W.MRG32K3A else "philox")
            parts[key] = {
                "ms": round(t_ms, 3), "Gsamples_per_s": round(N / (t_ms * 1e-3) / 1e9, 1),
                "Gnumbers_per_s": round(2 * N / (t_ms * 1e-3) / 1e9, 1), "hits": tot,
                "pi_hat": pi_hat, "within_4sigma": abs(pi_hat - math.pi) <= 4 * 4 * math.sqrt(p * (1 - p) / N),
                "scaling": "strong", "samples": N}
            # compute-bound (0 B per sample): issue roofline from the kernel's
            # instructions per sample (ncu, profiles/ncu_traffic.json) and the
            # time per sample measured here; per-pipe busy fractions beside it
            rec = profile_record(key.replace("mc_pi_", "mc_"))
            if rec and rec.get("inst_per_unit"):
                ach = rec["inst_per_unit"] * (N / world) / (t_ms * 1e-3)  # warp instructions / s
                parts[key]["roofline"] = {
                    "bound": "issue", "achieved": round(ach / 1e12, 4), "peak": round(ISSUE_PEAK / 1e12, 4),
                    "unit": "T warp instr/s", "frac": round(ach / ISSUE_PEAK, 4),
                    "warp_inst_per_sample": round(rec["inst_per_unit"], 4),
                    "peak_source": "148 SMs x 4 schedulers x 1 warp instr/clk x 1.965 GHz (B200_PROFILING.md)",
                    "pipes": {k: rec.get(k) for k in ("issue_active_pct", "fp64_pipe_pct", "fmaheavy_pipe_pct",
                                                      "alu_pipe_pct") if rec.get(k) is not None},
                    "limiter": limiter_from_profiles(key.replace("mc_pi_", "mc_"))}
            del st
        ws = W.rank_slice(shrink(W.C3), rank, world, weak=True)
        out64 = out.view(torch.float64)[: ws.n_streams * ws.n // 2]
        # 2^20 x 4096 f64 needs 32 GiB: fill half the rows per launch into the 16 GiB buffer
        half = ws.n_streams // 2
        times = []
        for it in range(4):
            h = shv.shv_streams_create_ex(ws.gen, list(ws.seed), ws.first, half, ws.spacing, state,
                                          0, local, sp)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            shv.shv_generate_f64(h, out64, ws.n, sp)
            b.record(stream)
            torch.cuda.synchronize()
            shv.shv_streams_destroy(h)
            if it:
                times.append(a.elapsed_time(b))
        t_ms = statistics.mean(times)
        parts["mrg_fill_f64"] = {"ms": round(t_ms, 4), "numbers": half * ws.n,
                                 "Gnumbers_per_s": round(half * ws.n / (t_ms * 1e-3) / 1e9, 1),
                                 "GB_per_s": round(8 * half * ws.n / (t_ms * 1e-3) / 1e9, 1),
                                 "frac_of_hbm_peak": round(8 * half * ws.n / (t_ms * 1e-3) / 1e9 / peak, 4)}

        def fill_ms(h, buf, nn, reps=3, kind="u32"):
            """Mean of `reps` launches after one untimed launch (events on the launching stream)."""
            gen = {"u32": shv.shv_generate_u32, "f64": shv.shv_generate_f64}[kind]
            times = []
            for it in range(reps + 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                gen(h, buf, nn, sp)
                b.record(stream)
                torch.cuda.synchronize()
                if it:
                    times.append(a.elapsed_time(b))
            return statistics.mean(times)

        def fill_part(t_ms, numbers, bpn=4):
            return {"ms": round(t_ms, 4), "Gnumbers_per_s": round(numbers / (t_ms * 1e-3) / 1e9, 1),
                    "GB_per_s": round(bpn * numbers / (t_ms * 1e-3) / 1e9, 1),
                    "frac_of_hbm_peak": round(bpn * numbers / (t_ms * 1e-3) / 1e9 / peak, 4)}

        # Threefry4x64-20 (NEXT-2) on the C5 shape: 2^20 counter-streams x 4096 u32
        h = shv.shv_streams_create_ex(W.THREEFRY4X64_20, [12345], wp.first, wp.n_streams, 0, None, 0,
                                      local, sp)
        parts["threefry_fill_u32"] = fill_part(fill_ms(h, out, n), total_per_rank)
        shv.shv_streams_destroy(h)
        # TinyMT32 (NEXT-3) on the C5 shape: 2^20 streams x 4096 u32, groups of 256
        # streams sharing a parameter set (test parameter sets, R15)
        ns_t = wm.n_streams
        params = W.tinymt32_test_params((wm.first + ns_t) // 256 + 1)
        st_t = torch.empty(4 * ns_t, dtype=torch.int32, device=dev)
        h = shv.shv_streams_create_tinymt32(params, 12345, 256, wm.first, ns_t, st_t, 0, local, sp)
        parts["tinymt_fill_u32"] = fill_part(fill_ms(h, out, n), total_per_rank)
        shv.shv_streams_destroy(h)
        del st_t

        # MTGP32-11213 (NEXT-4c, R18): the 200 parameter sets of the toolkit's DC
        # table, one CTA-cooperative state each, 2^32 / 200 u32 per stream
        try:
            mt_params = W.mtgp32_params()
        except FileNotFoundError:
            mt_params = None
        if mt_params:
            nmt = total_per_rank // len(mt_params)
            h = shv.shv_streams_create_mtgp32(mt_params, 12345, 0, len(mt_params), None, 0, local, sp)
            parts["mtgp32_fill_u32"] = {**fill_part(fill_ms(h, out, nmt), nmt * len(mt_params)),
                                        "streams": len(mt_params), "numbers_per_stream": nmt}
            shv.shv_streams_destroy(h)

        # Leap Frog (NEXT-4, R17) on the C5 shape: 2^20 players of one base
        # sequence x 4096 u32 per rank (rank r deals players [r*2^20, (r+1)*2^20)
        # of K = world*2^20)
        K = wm.n_streams * world
        for key, gen, seed in (("leapfrog_mrg_fill_u32", W.MRG32K3A, wm.seed),
                               ("leapfrog_philox_fill_u32", W.PHILOX4X32_10, wp.seed),
                               ("leapfrog_threefry_fill_u32", W.THREEFRY4X64_20, (12345,))):
            h = shv.shv_streams_create_leapfrog(gen, list(seed), K, rank * wm.n_streams, wm.n_streams,
                                                state if gen == W.MRG32K3A else None, 0, local, sp)
            parts[key] = fill_part(fill_ms(h, out, n), total_per_rank)
            shv.shv_streams_destroy(h)

        # Disjointness audit (NEXT-4; S L407-415) of the first 2^18 MRG32k3a C5
        # rows (2^18 x 4093 ~ 1.07e9 four-word windows, 34 GB hash table)
        na = min(wm.n_streams, 1 << 18)
        h = shv.shv_streams_create_ex(wm.gen, list(wm.seed), wm.first, na, wm.spacing, state, 0, local, sp)
        shv.shv_generate_u32(h, out, n, sp)
        shv.shv_streams_destroy(h)
        wsb = shv.shv_verify_disjoint_workspace_bytes(na, n)
        ws_a = torch.empty(wsb // 8, dtype=torch.int64, device=dev)
        rep = torch.zeros(7, dtype=torch.int64, device=dev)
        times = []
        for it in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            shv.shv_verify_disjoint(out, na, n, ws_a, wsb, rep, sp)
            b.record(stream)
            torch.cuda.synchronize()
            if it:
                times.append(a.elapsed_time(b))
        r = dict(zip(shv.DISJOINT_REPORT_FIELDS, rep.cpu().tolist()))
        t_ms = statistics.mean(times)
        parts["audit_mrg_c5_prefix"] = {"ms": round(t_ms, 3), "pe": na, "horizon": n, "windows": r["windows"],
                                        "Gwindows_per_s": round(r["windows"] / (t_ms * 1e-3) / 1e9, 2),
                                        "disjoint": bool(r["disjoint"]), "colliding": r["colliding"],
                                        "workspace_bytes": wsb}
        del ws_a

        # TinyMT32 Leap Frog (R19) on the C5 shape: K = world * 2^20 players of the
        # check parameter set's base sequence; each draw skips K - 1 base draws
        # with the GF(2) matrix T^(K-1)
        h = shv.shv_streams_create_leapfrog(W.TINYMT32, [12345, *W.TINYMT32_CHECK_PARAMS], K,
                                            rank * wm.n_streams, wm.n_streams, None, 0, local, sp)
        parts["leapfrog_tinymt_fill_u32"] = fill_part(fill_ms(h, out, n, reps=2), total_per_rank)
        shv.shv_streams_destroy(h)

        # C6: stream-count sweep at a fixed 2^32 u32 per GPU (16 GiB),
        # n_streams = 2^13 .. 2^22, n_per_stream = total / n_streams, both generators.
        # Acceptance: every point within 10% of the C5 (2^20 x 4096) figure.
        # Power-capped clocks drift with sustained load, so the points are timed
        # in three rounds, each in a shuffled order, and the median is kept.
        st_s = torch.empty(6 << 22, dtype=torch.int32, device=dev)
        points = [(key, lg) for lg in range(13, 23) for key in ("mrg", "philox")
                  if total_per_rank // (1 << lg) >= 8]
        samples = {p: [] for p in points}
        rng = random.Random(1234)
        for _ in range(3):
            rng.shuffle(points)
            for key, lg in points:
                ns = 1 << lg
                nn = total_per_rank // ns
                w = wm if key == "mrg" else wp
                h = shv.shv_streams_create_ex(w.gen, list(w.seed), rank * ns, ns, w.spacing,
                                              st_s if key == "mrg" else None, 0, local, sp)
                samples[(key, lg)].append(ns * nn / (fill_ms(h, out, nn, reps=2) * 1e-3) / 1e9)
                shv.shv_streams_destroy(h)
        del st_s
        sweep = {"mrg": {}, "philox": {}}
        for (key, lg), v in sorted(samples.items(), key=lambda kv: kv[0][1]):
            sweep[key][f"2^{lg}"] = round(statistics.median(v), 1)
        c5 = {k: parts[k]["Gnumbers_per_s"] for k in ("mrg", "philox")}
        ref = {k: v.get("2^20") for k, v in sweep.items()}  # same protocol as the other points
        parts["c6_stream_sweep"] = {
            "unit": "Gnumbers/s", "numbers_per_gpu": total_per_rank, **sweep, "c5_in_step": c5,
            "min_over_2^20": {k: round(min(v.values()) / ref[k], 3) for k, v in sweep.items() if v and ref[k]},
            "flat_within_10pct": all(min(v.values()) >= 0.9 * ref[k] for k, v in sweep.items() if v and ref[k]),
            "protocol": "each point: fresh handle, 1 untimed + 2 timed launches (CUDA events); 3 shuffled rounds, median"}

    # ---- e2e: same workload through shv_generate_u32_host into pinned host memory ----
    e2e = None
    if not args.no_e2e:
        # bounded pinned memory per rank: the rows go out in slices of at most
        # 2 GiB (2^17 streams), each slice a handle over its stream range
        # (first_stream) written into the same pinned buffer
        slice_streams = max(1, min(wm.n_streams, (2 << 30) // (4 * n)))
        host = torch.empty(slice_streams * n, dtype=torch.int32, pin_memory=True)
        e2e_steps = min(args.steps, 3)

        def step_host():
            for w, stt in ((wm, state), (wp, None)):
                for s0 in range(0, w.n_streams, slice_streams):
                    ns_ = min(slice_streams, w.n_streams - s0)
                    h = shv.shv_streams_create_ex(w.gen, list(w.seed), w.first + s0, ns_, w.spacing,
                                                  stt, 0, local, sp)
                    shv.shv_generate_u32_host(h, host, n, sp)
                    shv.shv_streams_destroy(h)
        step_host()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(e2e_steps):
            step_host()
        b.record(stream)
        barrier()
        e_ms = max_over_ranks(a.elapsed_time(b))
        e2e = {"value": 2 * total_per_rank * world * e2e_steps / (e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 2 * 4 * total_per_rank,
               "steps": e2e_steps, "api": "shv_generate_u32_host (pinned host buffer)",
               "pinned_bytes_per_rank": slice_streams * n * 4,
               "note": "inputs are seed words passed as call arguments; no input tensor is copied"}
        del host

    if rank == 0:
        cpu = None
        if not args.no_cpu:
            import oracle
            oracle.build()
            threads = len(os.sched_getaffinity(0))
            cpu = cpu_baseline(threads)
            if not args.no_parts:
                cpu["mc_pi"] = cpu_baseline_mc(threads)
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic",
                "config": {"workload": WORKLOAD, "streams_per_gpu": wm.n_streams,
                           "process_group": ({"backend": dist.get_backend(), "world": world}
                                             if launched else None),
                           "numbers_per_stream": n, "bytes_per_gpu_per_generator": alg_bytes,
                           "parallelism": f"streams sharded over {world} GPU(s), no data-path collective",
                           "l2": "no flush: each launch writes 16 GiB >> 126 MB L2"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": 3 * args.steps, "clocks": clk, "parts": parts,
                "per_gpu_Gnumbers_per_s": round(value / world, 2)}
        print(json.dumps(line), flush=True)
    if launched:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
