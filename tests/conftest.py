import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA library")
    config.addinivalue_line("markers", "slow: long-running oracle work")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


class CurandPin:
    """cuRAND's header implementations compiled as host code (tests/pins)."""

    def __init__(self, exe):
        self.p = subprocess.Popen([exe], stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                                  text=True, bufsize=1)

    def ask(self, *words):
        self.p.stdin.write(" ".join(str(w) for w in words) + "\n")
        self.p.stdin.flush()
        line = self.p.stdout.readline().split()
        assert line and line[0] != "error", words
        return [int(v) for v in line]

    def close(self):
        self.p.stdin.close()
        self.p.wait()


@pytest.fixture(scope="session")
def curand_pin(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available to build the cuRAND host pin")
    exe = str(tmp_path_factory.mktemp("pin") / "curand_host_pin")
    subprocess.check_call([nvcc, "-w", "-O1", "-o", exe,
                           os.path.join(ROOT, "tests", "pins", "curand_host_pin.cu")])
    pin = CurandPin(exe)
    yield pin
    pin.close()


@pytest.fixture(scope="session")
def mtgp_pin(tmp_path_factory):
    """cuRAND's MTGP32 (host-callable header code + the 11213 parameter sets)."""
    gxx = shutil.which("g++")
    inc = "/usr/local/cuda/include"
    if not gxx or not os.path.exists(os.path.join(inc, "curand_mtgp32dc_p_11213.h")):
        pytest.skip("g++ or the CUDA toolkit headers are not available for the MTGP32 pin")
    exe = str(tmp_path_factory.mktemp("mtgp") / "mtgp_host_pin")
    subprocess.check_call([gxx, "-w", "-O1", "-I", inc, "-o", exe,
                           os.path.join(ROOT, "tests", "pins", "mtgp_host_pin.cpp")])
    pin = CurandPin(exe)
    yield pin
    pin.close()
