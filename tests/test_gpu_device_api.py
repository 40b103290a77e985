"""The device-side API (include/shv_rng.cuh; P L387-399, Listing 1 P L480-499):
a user kernel constructs shv::Rng<GEN>(view, thread id) and calls next();
every value must equal the oracle's for that stream at the handle's offset."""
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
def listing1(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    so = str(tmp_path_factory.mktemp("l1") / "liblisting1.so")
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
                           "-o", so, os.path.join(ROOT, "tests", "gpu_kernels", "listing1.cu")])
    lib = C.CDLL(so)
    lib.launch_listing1.restype = C.c_int
    lib.launch_listing1.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
    return lib


DT = {0: (torch.int32, np.uint32), 1: (torch.float32, np.float32), 2: (torch.float64, np.float64)}


@pytest.mark.parametrize("gen,sp", [(W.MRG32K3A, W.SPACING_STREAM), (W.MRG32K3A, W.SPACING_SUBSTREAM),
                                    (W.PHILOX4X32_10, W.SPACING_STREAM),
                                    (W.PHILOX4X32_10, W.SPACING_KEYED), (W.THREEFRY4X64_20, W.SPACING_STREAM)])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_listing1_kernel_matches_oracle(shv, orc, listing1, gen, sp, kind):
    block_num, thread_num = 37, 128          # Listing 1: init(block_num); <<<block_num, thread_num>>>
    n = block_num * thread_num
    seed = [12345] if gen == W.MRG32K3A else ([777, 5, 6, 7] if gen == W.THREEFRY4X64_20 else [777])
    first = 5
    state = torch.empty(6 * n, dtype=torch.int32, device="cuda") if gen == W.MRG32K3A else None
    h = shv.shv_streams_create_ex(gen, seed, first, n, sp, state, 0, torch.cuda.current_device(), None)
    offset = 0
    for per_thread, jump in ((1, 0), (13, 3), (40, 0)):   # a Listing-1 call, then longer ones
        if jump:
            shv.shv_jump(h, shv.SHV_JUMP_DRAWS, jump)
            offset += jump
        torch.cuda.synchronize()
        v = shv.shv_get_device_view(h)
        tdt, ndt = DT[kind]
        out = torch.empty(n * per_thread, dtype=tdt, device="cuda")
        assert listing1.launch_listing1(gen, kind, out.data_ptr(), C.addressof(v), per_thread,
                                        block_num, thread_num) == 0
        got = out.cpu().numpy().view(ndt).reshape(n, per_thread)
        ref = orc.generate(gen, seed, n, per_thread, first=first, spacing=sp, offset=offset, kind=kind)
        bits = np.uint32 if got.itemsize == 4 else np.uint64  # compare bit patterns
        assert np.array_equal(got.view(bits), ref.view(bits))
        # the kernel consumed per_thread values per stream: advance the handle
        draws = per_thread * (2 if (kind == 2 and gen != W.MRG32K3A) else 1)
        shv.shv_jump(h, shv.SHV_JUMP_DRAWS, draws)
        offset += draws
    # the bulk path continues exactly where the device API left off
    out = torch.empty(n * 8, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, out, 8, None)
    torch.cuda.synchronize()
    ref = orc.generate(gen, seed, n, 8, first=first, spacing=sp, offset=offset)
    assert np.array_equal(out.cpu().numpy().view(np.uint32).reshape(n, 8), ref)
    shv.shv_streams_destroy(h)
