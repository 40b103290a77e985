"""TinyMT32 (NEXT-3; P L287-317 §4.2; R15) on the GPU against the oracle: the
paper's hybrid distribution (one parameter set per group, 2^64-draw slices per
stream inside a group), stateful generate/mc_pi, jumps (stepped and by the
jump polynomial, on the caller's stream), ragged shapes, and the device API."""
import ctypes as C
import os
import shutil
import subprocess

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DT = {"u32": (torch.int32, np.uint32, 0), "f32": (torch.float32, np.float32, 1),
      "f64": (torch.float64, np.float64, 2)}


@pytest.fixture(scope="module")
def shv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1412_8266_b200 as shv
    return shv


def bits(a):
    return a.view(np.uint32 if a.itemsize == 4 else np.uint64)


@pytest.mark.parametrize("kind", ["u32", "f32", "f64"])
@pytest.mark.parametrize("gs,first,ns", [(32, 0, 256), (8, 13, 70), (1, 3, 5), (256, 0, 1024)])
def test_tinymt_fill_replay_and_jump(shv, orc, kind, gs, first, ns):
    params = W.tinymt32_test_params((first + ns + gs - 1) // gs)
    sd = W.tinymt32_seed_words(4242, gs, params)
    h = shv.shv_streams_create_tinymt32(params, 4242, gs, first, ns, None, 0, -1, None)
    tdt, ndt, kid = DT[kind]
    dpv = 2 if kind == "f64" else 1
    off = 0
    for n, jump in ((64, 0), (13, 0), (512, 7), (8, 0)):
        if jump:
            shv.shv_jump(h, shv.SHV_JUMP_DRAWS, jump)
            off += jump
        out = torch.empty(ns * n, dtype=tdt, device="cuda")
        getattr(shv, "shv_generate_" + kind)(h, out, n, None)
        torch.cuda.synchronize()
        ref = orc.generate(W.TINYMT32, sd, ns, n, first=first, offset=off, kind=kid)
        assert np.array_equal(bits(out.cpu().numpy().view(ndt).reshape(ns, n)), bits(ref)), (n, jump)
        off += n * dpv
    assert shv.shv_get_position(h)["offset"] == off
    shv.shv_streams_destroy(h)


def test_tinymt_mc_counts(shv, orc):
    gs, ns = 64, 640
    params = W.tinymt32_test_params(ns // gs)
    sd = W.tinymt32_seed_words(7, gs, params)
    h = shv.shv_streams_create_tinymt32(params, 7, gs, 0, ns, None, 0, -1, None)
    hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(ns, dtype=torch.int64, device="cuda")
    shv.shv_mc_pi_ex(h, 3000, hits, cnt, None)
    torch.cuda.synchronize()
    tot, ref = orc.mc_count(W.TINYMT32, sd, ns, 3000)
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), ref) and int(hits.item()) == tot
    shv.shv_streams_destroy(h)


def test_tinymt_check_output_on_gpu(shv):
    rows = [ln.split() for ln in open(os.path.join(ROOT, "tests", "golden", "tinymt32_check.txt"))
            if ln.strip() and not ln.startswith("#")]
    m1, m2, tm, seed, *outs = rows[0]
    h = shv.shv_streams_create_tinymt32([(int(m1, 16), int(m2, 16), int(tm, 16))], int(seed), 1, 0, 1,
                                        None, 0, -1, None)
    out = torch.empty(10, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, out, 10, None)
    torch.cuda.synchronize()
    assert out.cpu().numpy().view(np.uint32).tolist() == [int(v) for v in outs]
    shv.shv_streams_destroy(h)


def test_tinymt_device_api(shv, orc, tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    so = str(tmp_path / "liblisting1.so")
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
                           "-DWITH_TINYMT", "-o", so, os.path.join(ROOT, "tests", "gpu_kernels", "listing1.cu")])
    lib = C.CDLL(so)
    lib.launch_listing1.restype = C.c_int
    lib.launch_listing1.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
    gs, blocks, threads = 128, 8, 128
    n = blocks * threads
    params = W.tinymt32_test_params(n // gs)
    h = shv.shv_streams_create_tinymt32(params, 31, gs, 0, n, None, 0, -1, None)
    v = shv.shv_get_device_view(h)
    out = torch.empty(n * 9, dtype=torch.int32, device="cuda")
    assert lib.launch_listing1(W.TINYMT32, 0, out.data_ptr(), C.addressof(v), 9, blocks, threads) == 0
    ref = orc.generate(W.TINYMT32, W.tinymt32_seed_words(31, gs, params), n, 9)
    assert np.array_equal(out.cpu().numpy().view(np.uint32).reshape(n, 9), ref)
    shv.shv_streams_destroy(h)


@pytest.mark.parametrize("gs,first,ns", [(32, 0, 256), (8, 13, 70), (1, 3, 5)])
def test_tinymt_polynomial_jumps(shv, orc, gs, first, ns):
    """Jumps past the stepping threshold use x^n mod the minimal polynomial of
    each parameter set's orbit (shv_api.cpp shv_jump): any n, compared with
    the oracle's GF(2) matrix power (orc_tinymt32_jump)."""
    params = W.tinymt32_test_params((first + ns + gs - 1) // gs)
    sd = W.tinymt32_seed_words(99, gs, params)
    h = shv.shv_streams_create_tinymt32(params, 99, gs, first, ns, None, 0, -1, None)
    off = 0
    for jump in (257, 1000, (1 << 33) + 5, (1 << 63) + 12345, 256, 1):
        shv.shv_jump(h, shv.SHV_JUMP_DRAWS, jump)
        off += jump
        out = torch.empty(ns * 40, dtype=torch.int32, device="cuda")
        shv.shv_generate_u32(h, out, 40, None)
        torch.cuda.synchronize()
        ref = orc.generate(W.TINYMT32, sd, ns, 40, first=first, offset=off)
        assert np.array_equal(out.cpu().numpy().view(np.uint32).reshape(ns, 40), ref), jump
        off += 40
    shv.shv_streams_destroy(h)


def test_tinymt_jump_on_callers_stream(shv, orc):
    """Create on stream A, jump on stream B, generate on stream C; the caller
    orders the streams with events. The state advance runs on B."""
    gs, ns = 16, 128
    params = W.tinymt32_test_params(ns // gs)
    sd = W.tinymt32_seed_words(5, gs, params)
    sa, sb, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    h = shv.shv_streams_create_tinymt32(params, 5, gs, 0, ns, None, 0, -1, sa)
    sb.wait_stream(sa)
    for jump in (100, 1 << 40):  # stepped, polynomial
        shv.shv_jump(h, shv.SHV_JUMP_DRAWS, jump, sb)
    sc.wait_stream(sb)
    out = torch.empty(ns * 64, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, out, 64, sc)
    sc.synchronize()
    ref = orc.generate(W.TINYMT32, sd, ns, 64, offset=100 + (1 << 40))
    assert np.array_equal(out.cpu().numpy().view(np.uint32).reshape(ns, 64), ref)
    shv.shv_streams_destroy(h)
