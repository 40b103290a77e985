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


def test_single_rank_bench_contract_small():
    """The one JSON line of the default (N = 1) bench path, small shapes: every
    key of the contract, the binding roofline with the HBM figure beside it,
    the oracle baseline and the end-to-end figure through host buffers."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--small"], cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["dtype"] == "u32"
    assert "workload" in d["config"] and d["gpu_launches"] == 3 * 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] and r["achieved"] > 0 and r["peak"] > 0
    assert r["algorithmic_bytes_per_launch"] == 4 * (1 << 14) * 4096
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert c["single_thread"]["cores"] == 1 and c["single_thread"]["value"] > 0
    m = c["mc_pi"]
    assert m["kind"] == "oracle" and m["unit"] == "Gsamples/s" and m["value"] > 0 and m["single_thread"]["cores"] == 1
    for key in ("mc_pi_mrg", "mc_pi_philox"):
        assert d["parts"][key]["within_4sigma"] in (True, False)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_nccl_bench_path_one_rank(orc):
    """torchrun with one rank and the NCCL backend: the process group, the
    device-bound NCCL communicator and the Monte Carlo all_reduce run (the
    SCALE path on a one-GPU box); NCCL_DEBUG=INFO shows the library loaded."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "1",
           "--steps", "3", "--warmup", "3", "--small", "--backend", "nccl", "--no-e2e", "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["process_group"] == {"backend": "nccl", "world": 1}
    assert "nccl version" in (out.stderr + out.stdout).lower()  # NCCL_DEBUG=INFO: the library initialised
    for key, w in (("mc_pi_mrg", W.C4_MRG), ("mc_pi_philox", W.C4_PHILOX)):
        tot, _ = orc.mc_count(w.gen, list(w.seed), 1 << 14, 1 << 12, spacing=w.spacing)
        assert d["parts"][key]["hits"] == tot, key
