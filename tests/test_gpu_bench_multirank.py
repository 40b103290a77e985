"""The N>1 bench path end to end on the GPU box: two ranks under torchrun
(sharing one GPU, gloo process group, as NCCL needs one GPU per rank), small
shapes. Checks the one JSON line and that the Monte Carlo totals after the
cross-rank all_reduce equal the oracle's single-process totals (SURVEY §8e:
bit-identical for every world size)."""
import json
import os
import socket
import subprocess
import sys

import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_bench_small(orc):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--small", "--backend", "gloo", "--no-e2e", "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] == 3 * 3
    for key, w in (("mc_pi_mrg", W.C4_MRG), ("mc_pi_philox", W.C4_PHILOX)):
        ns, samples = 1 << 14, 1 << 12
        tot, _ = orc.mc_count(w.gen, list(w.seed), ns, samples, spacing=w.spacing)
        assert d["parts"][key]["hits"] == tot, key
