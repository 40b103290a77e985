"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/shv.h declares, and its host-only logic (validation, lifecycle errors,
partitioner, host-built jump matrices) is right. No compute calls here."""
import os
import random
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shv.h")


@pytest.fixture(scope="module")
def shv():
    from paper_1412_8266_b200 import _build
    _build.build()
    import paper_1412_8266_b200 as shv
    return shv


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\**(shv_[a-z_0-9]+)\(", txt, re.M)))


def test_header_symbols_exported(shv):
    declared = _declared()
    assert len(declared) >= 15
    out = subprocess.check_output(["nm", "-D", "--defined-only", shv.LIB_PATH], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert sorted(shv.EXPORTS) == declared


def test_library_is_sm100a(shv):
    out = subprocess.check_output(["cuobjdump", "--list-elf", shv.LIB_PATH], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", shv.LIB_PATH], text=True)
    assert "STG.E.ENL2.256" in sass  # 32-byte vector stores (sm_100+ only)
    assert "HMMA" not in sass and "UTCHMMA" not in sass  # not a contraction
    assert "shv 0.1 sm_100a" == shv.shv_build_info()


def test_status_strings(shv):
    for code in range(10):
        assert shv.shv_status_string(code).startswith("SHV_")


def test_validation_errors_without_gpu(shv):
    E = shv.ShvError
    cases = [
        (dict(gen=shv.SHV_GEN_MRG32K3A, seed=[0] * 6), shv.SHV_ERR_INVALID_SEED),
        (dict(gen=shv.SHV_GEN_MRG32K3A, seed=[1, 1, 1, 0, 0, 0]), shv.SHV_ERR_INVALID_SEED),
        (dict(gen=shv.SHV_GEN_MRG32K3A, seed=[4294967087] + [1] * 5), shv.SHV_ERR_INVALID_SEED),
        (dict(gen=shv.SHV_GEN_MRG32K3A, seed=[1, 2]), shv.SHV_ERR_INVALID_ARGUMENT),
        (dict(gen=shv.SHV_GEN_PHILOX4X32_10, seed=[1, 2, 3]), shv.SHV_ERR_INVALID_ARGUMENT),
        (dict(gen=7, seed=[1]), shv.SHV_ERR_INVALID_ARGUMENT),
        (dict(gen=shv.SHV_GEN_MRG32K3A, seed=[5], n_streams=0), shv.SHV_ERR_INVALID_ARGUMENT),
        (dict(gen=shv.SHV_GEN_PHILOX4X32_10, seed=[5], spacing=1), shv.SHV_ERR_UNSUPPORTED),
        (dict(gen=shv.SHV_GEN_MRG32K3A, seed=[5], spacing=1, first=(1 << 51) - 3, n_streams=4),
         shv.SHV_ERR_INSUFFICIENT_STREAMS),
        (dict(gen=shv.SHV_GEN_PHILOX4X32_10, seed=[5], first=(1 << 64) - 3, n_streams=4),
         shv.SHV_ERR_INSUFFICIENT_STREAMS),
        (dict(gen=shv.SHV_GEN_MRG32K3A, seed=[5], spacing=9), shv.SHV_ERR_INVALID_ARGUMENT),
        # keyed Philox (Parameterization): MRG has no keys; one tag word; ids < 2^32
        (dict(gen=shv.SHV_GEN_MRG32K3A, seed=[5], spacing=2), shv.SHV_ERR_UNSUPPORTED),
        (dict(gen=shv.SHV_GEN_PHILOX4X32_10, seed=[5, 6], spacing=2), shv.SHV_ERR_INVALID_ARGUMENT),
        (dict(gen=shv.SHV_GEN_PHILOX4X32_10, seed=[5], spacing=2, first=(1 << 32) - 3, n_streams=4),
         shv.SHV_ERR_INSUFFICIENT_STREAMS),
    ]
    for kw, code in cases:
        with pytest.raises(E) as ei:
            shv.shv_streams_create_ex(kw["gen"], kw["seed"], kw.get("first", 0),
                                      kw.get("n_streams", 8), kw.get("spacing", 0), None, 0, 0, 0)
        assert ei.value.status == code, kw


def test_tinymt32_validation_without_gpu(shv):
    E = shv.ShvError
    P = [(0x8F7011EE, 0xFC78FF1F, 0x3793FDFF)] * 2
    for args, code in (((None, 1, 4, 0, 8), shv.SHV_ERR_MISSING_PARAMETERS),
                       (([], 1, 4, 0, 8), shv.SHV_ERR_MISSING_PARAMETERS),
                       ((P, 1, 4, 0, 9), shv.SHV_ERR_INSUFFICIENT_STREAMS),   # 3 groups, 2 sets
                       ((P, 1, 3, 0, 4), shv.SHV_ERR_INVALID_ARGUMENT),      # not a power of two
                       ((P, 1, 4, 0, 0), shv.SHV_ERR_INVALID_ARGUMENT)):
        params, seed, gs, first, n = args
        with pytest.raises(E) as ei:
            shv.shv_streams_create_tinymt32(params or [], seed, gs, first, n, None, 0, 0, 0)
        assert ei.value.status == code, args
    with pytest.raises(E) as ei:  # the generic create does not make TinyMT handles
        shv.shv_streams_create_ex(shv.SHV_GEN_TINYMT32, [1], 0, 4, 0, None, 0, 0, 0)
    assert ei.value.status == shv.SHV_ERR_MISSING_PARAMETERS
    assert shv.shv_state_bytes(shv.SHV_GEN_TINYMT32, 10) == 160


def test_lifecycle_errors_without_gpu(shv):
    for fn in (lambda: shv.shv_streams_destroy(123456789),
               lambda: shv.shv_jump(123456789, 0, 1, 0),
               lambda: shv.shv_get_position(123456789),
               lambda: shv.shv_generate_u32(123456789, 0, 8, 0),
               lambda: shv.shv_mc_pi(123456789, 8, 0, 0),
               lambda: shv.shv_set_launch_config(123456789)):
        with pytest.raises(shv.ShvError) as ei:
            fn()
        assert ei.value.status == shv.SHV_ERR_LIFECYCLE
    assert shv.shv_state_bytes(shv.SHV_GEN_MRG32K3A, 1 << 20) == 24 << 20
    assert shv.shv_state_bytes(shv.SHV_GEN_PHILOX4X32_10, 1 << 20) == 0


def test_partition_covers_disjointly(shv):
    for total in (1, 7, 1 << 20, (1 << 64) - 1):
        for world in (1, 2, 3, 4, 8):
            nxt = 0
            for r in range(world):
                f, c = shv.shv_partition(total, r, world)
                assert f == nxt
                nxt = f + c
            assert nxt == total
    with pytest.raises(shv.ShvError):
        shv.shv_partition(10, 2, 2)


def test_host_jump_matrices_match_oracle(shv, orc):
    A1, A2 = orc.mrg_matrices()
    rng = random.Random(9)
    exps = [0, 1, 2, 3, 1 << 76, 1 << 127, (1 << 128) - 1] + [rng.getrandbits(128) for _ in range(60)]
    for e in exps:
        a, b = shv.shv_jump_matrix(e)
        assert a == orc.mat_pow(A1, e, orc.M1), e
        assert b == orc.mat_pow(A2, e, orc.M2), e


def test_product_does_not_touch_oracle():
    # The product package and its sources never reference the oracle.
    pkg = os.path.join(ROOT, "paper_1412_8266_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.lower().replace("no cpu fallback", ""), f


def test_leapfrog_validation_without_gpu(shv):
    # Leap Frog handles (R17): rejected before any CUDA call
    E = shv.ShvError
    for args, code in (((shv.SHV_GEN_TINYMT32, [1], 4, 0, 4), shv.SHV_ERR_MISSING_PARAMETERS),  # R19: 4 words
                       ((shv.SHV_GEN_MTGP32, [1], 4, 0, 4), shv.SHV_ERR_UNSUPPORTED),
                       ((shv.SHV_GEN_PHILOX4X32_10, [1], 0, 0, 4), shv.SHV_ERR_INVALID_ARGUMENT),
                       ((shv.SHV_GEN_PHILOX4X32_10, [1], 4, 0, 0), shv.SHV_ERR_INVALID_ARGUMENT),
                       ((shv.SHV_GEN_PHILOX4X32_10, [1], 4, 2, 3), shv.SHV_ERR_INSUFFICIENT_STREAMS),
                       ((shv.SHV_GEN_MRG32K3A, [1], (1 << 64) - 1, (1 << 64) - 2, 2),
                        shv.SHV_ERR_INSUFFICIENT_STREAMS),
                       ((shv.SHV_GEN_MRG32K3A, [0] * 6, 4, 0, 4), shv.SHV_ERR_INVALID_SEED),
                       ((shv.SHV_GEN_THREEFRY4X64_20, [1] * 5, 4, 0, 4), shv.SHV_ERR_INVALID_ARGUMENT)):
        with pytest.raises(E) as ei:
            shv.shv_streams_create_leapfrog(*args, None, 0, 0, 0)
        assert ei.value.status == code, args


def test_audit_workspace_size_without_gpu(shv):
    """shv_verify_disjoint_workspace_bytes (host-only): 8 * (6 + 5 * nb + 6 * W)
    for W = n_pe * (horizon - 3) windows, nb = 2^lg buckets with lg the
    smallest value (<= 11) for which W < 2^(17 + lg), i.e. >= ~2^16 windows
    per bucket; 0 when there are no windows or the codes
    would not fit in 40 bits."""
    def expect(n_pe, horizon):
        w = n_pe * (horizon - 3) if horizon >= 4 else 0
        if w == 0:
            return 0
        lg = 0
        while lg < 11 and (w >> (16 + lg)) > 0:
            lg += 1
        return 8 * (6 + 5 * (1 << lg) + 6 * w)
    for n_pe, horizon in ((1, 4), (2, 10), (8, 300), (1, 1 << 16), (256, 515), (1 << 18, 4096), (1 << 20, 4096),
                          (3, 2), (0, 100)):
        assert shv.shv_verify_disjoint_workspace_bytes(n_pe, horizon) == expect(n_pe, horizon), (n_pe, horizon)
    assert shv.shv_verify_disjoint_workspace_bytes(1 << 20, 1 << 21) == 0
    # no windows: a valid call that needs no rows or workspace; the report is
    # written on the device, so only argument validation runs here
    with pytest.raises(shv.ShvError) as e:
        shv.shv_verify_disjoint(None, 1, 10, None, 0, None, 0)
    assert e.value.status == shv.SHV_ERR_INVALID_ARGUMENT
    with pytest.raises(shv.ShvError) as e:
        shv.shv_verify_disjoint(None, 1, 10, None, 0, 12, 0)  # misaligned report pointer
    assert e.value.status == shv.SHV_ERR_MISALIGNED
