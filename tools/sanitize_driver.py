"""Small-shape driver for compute-sanitizer: exercises every
kernel of libshv once (vector and scalar fill paths, all output kinds, fused
MC, seeding, TinyMT32 preparation, Leap Frog, MTGP32, the disjointness
audit) so memcheck / racecheck / synccheck /
initcheck see each of them.   compute-sanitizer --tool memcheck python tools/sanitize_driver.py

SHV_SAN_PART=nohost skips the shv_generate_u32_host calls, SHV_SAN_PART=host runs
only them (tools/sanitize.sh: initcheck cannot see the TMA bulk-tensor stores that
fill the host path's device staging slices, so the host part runs under initcheck
with --check-api-memory-access no, and this driver checks every staged value
against the same values generated into device memory)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_8266_b200 as shv  # noqa: E402
import workloads as W  # noqa: E402


PART = os.environ.get("SHV_SAN_PART", "all")


def host_part(dev):
    """shv_generate_u32_host for each generator family; every value must equal
    the device-memory fill of an identical handle (no stale staging word)."""
    ns, n = 300, 4096
    for gen, sp, seed in ((W.MRG32K3A, 1, [12345]), (W.PHILOX4X32_10, 0, [5, 6]), (W.THREEFRY4X64_20, 0, [1, 2, 3])):
        hs = []
        for _ in range(2):
            st = torch.empty(6 * ns, dtype=torch.int32, device="cuda") if gen == W.MRG32K3A else None
            hs.append((shv.shv_streams_create_ex(gen, seed, 11, ns, sp, st, 0, dev, None), st))
        host = torch.full((ns * n,), -1, dtype=torch.int32, pin_memory=True)
        shv.shv_generate_u32_host(hs[0][0], host, n, None)
        out = torch.empty(ns * n, dtype=torch.int32, device="cuda")
        shv.shv_generate_u32(hs[1][0], out, n, None)
        torch.cuda.synchronize()
        assert torch.equal(host, out.cpu()), f"host output differs from device output (gen {gen})"
        for h, _ in hs:
            shv.shv_streams_destroy(h)
    print("host part: staged values equal the device fill")


def run():
    dev = torch.cuda.current_device()
    if PART == "host":
        host_part(dev)
        print("sanitize driver done")
        return
    ns = 300
    for gen, sp, seed in ((W.MRG32K3A, 1, [12345]), (W.MRG32K3A, 0, [7]), (W.PHILOX4X32_10, 0, [5, 6]),
                          (W.PHILOX4X32_10, 2, [9]), (W.THREEFRY4X64_20, 0, [1, 2, 3])):
        st = torch.empty(6 * ns, dtype=torch.int32, device="cuda") if gen == W.MRG32K3A else None
        h = shv.shv_streams_create_ex(gen, seed, 11, ns, sp, st, 0, dev, None)
        for n in (64, 13):                      # vector path, scalar/generic path
            for dt, fn in ((torch.int32, shv.shv_generate_u32), (torch.float32, shv.shv_generate_f32),
                           (torch.float64, shv.shv_generate_f64)):
                out = torch.empty(ns * n, dtype=dt, device="cuda")
                fn(h, out, n, None)
        shv.shv_jump(h, shv.SHV_JUMP_DRAWS, 3)  # unaligned offsets: generic kernels
        out = torch.empty(ns * 64, dtype=torch.int32, device="cuda")
        shv.shv_generate_u32(h, out, 64, None)
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(ns, dtype=torch.int64, device="cuda")
        shv.shv_mc_pi_ex(h, 501, hits, cnt, None)
        if PART == "all":
            host = torch.empty(ns * 64, dtype=torch.int32, pin_memory=True)
            shv.shv_generate_u32_host(h, host, 64, None)
        torch.cuda.synchronize()
        shv.shv_streams_destroy(h)
    params = W.tinymt32_test_params(20)
    h = shv.shv_streams_create_tinymt32(params, 3, 16, 5, ns, None, 0, dev, None)
    for n in (64, 13):
        for dt, fn in ((torch.int32, shv.shv_generate_u32), (torch.float64, shv.shv_generate_f64)):
            out = torch.empty(ns * n, dtype=dt, device="cuda")
            fn(h, out, n, None)
    shv.shv_jump(h, shv.SHV_JUMP_DRAWS, 5)
    hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    shv.shv_mc_pi(h, 100, hits, None)
    torch.cuda.synchronize()
    shv.shv_streams_destroy(h)
    # Leap Frog players (MRG recurrence, Philox per-player and grouped, Threefry)
    for gen, seed, K, first in ((W.MRG32K3A, [12345], 77, 5), (W.PHILOX4X32_10, [5], 77, 5),
                                (W.PHILOX4X32_10, [5], 76, 5), (W.PHILOX4X32_10, [5], 80, 8),
                                (W.THREEFRY4X64_20, [1, 2], 77, 5), (W.THREEFRY4X64_20, [1, 2], 80, 8)):
        st = torch.empty(6 * 70, dtype=torch.int32, device="cuda") if gen == W.MRG32K3A else None
        h = shv.shv_streams_create_leapfrog(gen, seed, K, first, 70, st, 0, dev, None)
        for n in (64, 13):
            for dt, fn in ((torch.int32, shv.shv_generate_u32), (torch.float64, shv.shv_generate_f64)):
                out = torch.empty(70 * n, dtype=dt, device="cuda")
                fn(h, out, n, None)
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(70, dtype=torch.int64, device="cuda")
        shv.shv_mc_pi_ex(h, 101, hits, cnt, None)
        torch.cuda.synchronize()
        shv.shv_streams_destroy(h)
    # MRG32k3a row-tile fill (mrg_fill_rows_kernel): forced at a small shape by a
    # 1-block x 32-thread grid; nseg 32 and nseg 3 (tiles spanning rows, ragged)
    for ns_, n in ((600, 4096), (3201, 384), (64, 256 * 32 * 5)):  # S 128 nseg 32; S 128 nseg 3; run mode (10 tiles per row)
        st = torch.empty(6 * ns_, dtype=torch.int32, device="cuda")
        h = shv.shv_streams_create_ex(W.MRG32K3A, [12345], 3, ns_, 1, st, 0, dev, None)
        shv.shv_set_launch_config(h, 1, 32, 0)
        for dt, fn in ((torch.int32, shv.shv_generate_u32), (torch.float32, shv.shv_generate_f32)):
            out = torch.empty(ns_ * n, dtype=dt, device="cuda")
            fn(h, out, n, None)
        torch.cuda.synchronize()
        shv.shv_streams_destroy(h)
    # TinyMT32 Leap Frog (stepping and matrix skips)
    for K in (5, 70):
        h = shv.shv_streams_create_leapfrog(W.TINYMT32, [3, *W.TINYMT32_CHECK_PARAMS], K, 1, 4, None, 0, dev, None)
        for dt, fn in ((torch.int32, shv.shv_generate_u32), (torch.float64, shv.shv_generate_f64)):
            out = torch.empty(4 * 13, dtype=dt, device="cuda")
            fn(h, out, 13, None)
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        shv.shv_mc_pi(h, 7, hits, None)
        torch.cuda.synchronize()
        shv.shv_streams_destroy(h)
    # MTGP32-11213 (block-cooperative ring kernel)
    mp = W.mtgp32_params(12)
    h = shv.shv_streams_create_mtgp32(mp, 3, 2, 10, None, 0, dev, None)
    for n in (700, 13):
        for dt, fn in ((torch.int32, shv.shv_generate_u32), (torch.float32, shv.shv_generate_f32),
                       (torch.float64, shv.shv_generate_f64)):
            out = torch.empty(10 * n, dtype=dt, device="cuda")
            fn(h, out, n, None)
    shv.shv_jump(h, shv.SHV_JUMP_DRAWS, 1001)
    hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(10, dtype=torch.int64, device="cuda")
    shv.shv_mc_pi_ex(h, 333, hits, cnt, None)
    torch.cuda.synchronize()
    shv.shv_streams_destroy(h)
    # disjointness audit (hash table in the workspace)
    rows = torch.randint(0, 3, (8 * 300,), dtype=torch.int32, device="cuda")
    wsb = shv.shv_verify_disjoint_workspace_bytes(8, 300)
    ws = torch.empty(wsb // 8, dtype=torch.int64, device="cuda")
    rep = torch.zeros(7, dtype=torch.int64, device="cuda")
    shv.shv_verify_disjoint(rows, 8, 300, ws, wsb, rep, None)
    torch.cuda.synchronize()
    print("sanitize driver done")


if __name__ == "__main__":
    run()
