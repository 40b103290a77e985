"""Independent device cross-check: libshv's GPU rows against NVIDIA cuRAND's
own device implementations compiled for sm_100a (tests/gpu_kernels/
curand_device_pin.cu). The parity bar is the oracle (test_gpu_parity.py);
this adds a second, library-side witness on the same hardware: MRG32k3a
substreams (C3 layout, R4) and Philox4x32-10 counter-streams (C2 layout,
R6 = cuRAND's curand_init(seed, subsequence, offset)), bit-exact."""
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


@pytest.fixture(scope="module")
def shv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1412_8266_b200 as shv
    return shv


@pytest.fixture(scope="module")
def cur(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    so = str(tmp_path_factory.mktemp("cur") / "libcurand_pin.so")
    subprocess.check_call([nvcc, "-w", "-O2", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "-o", so,
                           os.path.join(ROOT, "tests", "gpu_kernels", "curand_device_pin.cu")])
    L = C.CDLL(so)
    L.curand_mrg_rows.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int, C.c_int, C.POINTER(C.c_uint32)]
    L.curand_philox_rows.argtypes = [C.c_void_p, C.c_ulonglong, C.c_ulonglong, C.c_ulonglong, C.c_int, C.c_int]
    return L


def u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("first,ns,n", [(0, 4096, 1024), ((1 << 20) - 37, 37, 4096), (123456789, 64, 520)])
def test_mrg32k3a_substreams_equal_curand_device(shv, cur, first, ns, n):
    st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
    h = shv.shv_streams_create_ex(W.MRG32K3A, [12345], first, ns, W.SPACING_SUBSTREAM, st, 0,
                                  torch.cuda.current_device(), None)
    ours = torch.empty(ns * n, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, ours, n, None)
    torch.cuda.synchronize()
    shv.shv_streams_destroy(h)
    ref = torch.empty(ns * n, dtype=torch.int32, device="cuda")
    seed6 = (C.c_uint32 * 6)(*([12345] * 6))
    assert cur.curand_mrg_rows(ref.data_ptr(), first, ns, n, seed6) == 0
    assert np.array_equal(u32(ours), u32(ref))


@pytest.mark.parametrize("first,ns,n,offset", [(0, 1 << 16, 1024, 0), (1 << 40, 100, 333, 0), (5, 64, 256, 7)])
def test_philox_counter_streams_equal_curand_device(shv, cur, first, ns, n, offset):
    h = shv.shv_streams_create_ex(W.PHILOX4X32_10, [12345], first, ns, W.SPACING_STREAM, None, 0,
                                  torch.cuda.current_device(), None)
    if offset:
        shv.shv_jump(h, shv.SHV_JUMP_DRAWS, offset)
    ours = torch.empty(ns * n, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, ours, n, None)
    torch.cuda.synchronize()
    shv.shv_streams_destroy(h)
    ref = torch.empty(ns * n, dtype=torch.int32, device="cuda")
    assert cur.curand_philox_rows(ref.data_ptr(), 12345, first, offset, ns, n) == 0
    assert np.array_equal(u32(ours), u32(ref))
