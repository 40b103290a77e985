"""Multi-process (gloo, world_size 2 and 4, CPU) coverage of the N>1 path's host
logic: the rank -> stream-range partitioner (C ABI shv_partition and
workloads.rank_slice, which bench.py uses), and the one collective of the path,
the all_reduce(SUM) of Monte Carlo hit counts. The per-rank
compute is done by the oracle here (no GPU); the invariants are the ones the
GPU run relies on: the union of rank outputs equals the 1-rank output and the
MC total is identical for every world size."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_1412_8266_b200 as shv
    import workloads as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total_streams, samples = 96, 500
    first, count = shv.shv_partition(total_streams, rank, world)
    ws = W.rank_slice(W.Workload("t", W.MRG32K3A, (12345,), total_streams, samples,
                                 W.SPACING_SUBSTREAM), rank, world, weak=False)
    assert (ws.first, ws.n_streams) == (first, count)
    res = {}
    for gen, sp in ((W.MRG32K3A, 1), (W.PHILOX4X32_10, 0)):
        hits, counts = oracle.mc_count(gen, [12345], count, samples, first=first, spacing=sp,
                                       nthreads=1)
        t = torch.tensor([hits], dtype=torch.int64)
        dist.all_reduce(t)  # the path's only collective
        rows = torch.from_numpy(oracle.generate(gen, [12345], count, 16, first=first, spacing=sp,
                                                nthreads=1).astype(np.int64))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([count], dtype=torch.int64))
        mx = int(max(s.item() for s in sizes))
        pad = torch.zeros(mx, 16, dtype=torch.int64)
        pad[:count] = rows
        gathered = [torch.zeros(mx, 16, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, pad)
        full = torch.cat([g[: int(s.item())] for g, s in zip(gathered, sizes)])
        res[gen] = (int(t.item()), full.numpy())
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(res)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_equals_single(world, orc):
    import workloads as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for gen, sp in ((W.MRG32K3A, 1), (W.PHILOX4X32_10, 0)):
        tot, _ = orc.mc_count(gen, [12345], 96, 500, spacing=sp)
        rows = orc.generate(gen, [12345], 96, 16, spacing=sp)
        assert res[gen][0] == tot
        assert np.array_equal(res[gen][1].astype(np.uint32), rows)


def test_weak_slices_are_disjoint_and_adjacent():
    import workloads as W
    for world in (1, 2, 4, 8):
        prev_end = 0
        for r in range(world):
            s = W.rank_slice(W.C5_MRG, r, world, weak=True)
            assert s.first == prev_end and s.n_streams == 1 << 20
            prev_end = s.first + s.n_streams
        assert prev_end <= 1 << 51  # substream index space (R4)
