"""GPU parity for Leap Frog handles (NEXT-4; P L118-122 [§2.3]; R17).

The sm_100a kernels (MRG32k3a stepped by the characteristic-polynomial
recurrence of A^K, counter-based generators by direct indexing) against the
oracle, which deals the base sequence by plain stepping and jumping
(oracle/shv_oracle.c orc_stream_open_leapfrog). Bit-exact for every kind.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

L = W.SPACING_LEAPFROG
GENS = {"mrg": (W.MRG32K3A, [12345]), "philox": (W.PHILOX4X32_10, [12345, 678]),
        "threefry": (W.THREEFRY4X64_20, [1, 2, 3, 4])}
DT = {"u32": (torch.int32, np.uint32, 0), "f32": (torch.float32, np.float32, 1),
      "f64": (torch.float64, np.float64, 2)}


@pytest.fixture(scope="module")
def shv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1412_8266_b200 as shv
    return shv


class Players:
    def __init__(self, shv, gen, seed, players, first, n):
        self.shv, self.gen, self.seed, self.K, self.first, self.n = shv, gen, seed, players, first, n
        self.state = torch.empty(6 * n, dtype=torch.int32, device="cuda") if gen == W.MRG32K3A else None
        self.h = shv.shv_streams_create_leapfrog(gen, seed, players, first, n, self.state, 0,
                                                 torch.cuda.current_device(), None)
        self.offset = 0

    def gen_(self, m, kind="u32", host=False):
        tdt, ndt, _ = DT[kind]
        if host:
            out = torch.empty(self.n * m, dtype=tdt, pin_memory=True)
            self.shv.shv_generate_u32_host(self.h, out, m, None)
        else:
            out = torch.empty(self.n * m, dtype=tdt, device="cuda")
            getattr(self.shv, "shv_generate_" + kind)(self.h, out, m, None)
        torch.cuda.synchronize()
        self.offset += m * (2 if kind == "f64" and self.gen != W.MRG32K3A else 1)
        return out.cpu().numpy().view(ndt).reshape(self.n, m)

    def ref(self, orc, m, kind="u32", streams=None, offset=None):
        return orc.generate(self.gen, self.seed, self.n, m, first=self.first, spacing=L,
                            players=self.K, offset=self.offset if offset is None else offset,
                            kind=DT[kind][2], streams=streams)

    def close(self):
        self.shv.shv_streams_destroy(self.h)


def same(a, b):
    assert a.shape == b.shape
    if a.dtype.kind == "f":
        a = a.view(np.uint32 if a.itemsize == 4 else np.uint64)
        b = b.view(a.dtype)
    bad = np.nonzero(a != b)
    assert len(bad[0]) == 0, f"{len(bad[0])} mismatches, first at {[x[:5] for x in bad]}"


@pytest.mark.parametrize("g", list(GENS))
@pytest.mark.parametrize("kind", ["u32", "f32", "f64"])
@pytest.mark.parametrize("K,first,n,m", [(1, 0, 1, 1000), (3, 0, 3, 1000), (1000, 17, 300, 1024), (1000, 16, 300, 1000), (1024, 8, 300, 520),
                                         ((1 << 40) + 7, (1 << 39) + 5, 256, 520)])
def test_leapfrog_fill_matches_oracle(shv, orc, g, kind, K, first, n, m):
    gen, seed = GENS[g]
    p = Players(shv, gen, seed, K, first, n)
    try:
        for _ in range(2):  # second call continues at the advanced offset
            ref = p.ref(orc, m, kind)
            same(p.gen_(m, kind), ref)
    finally:
        p.close()


@pytest.mark.parametrize("g", list(GENS))
@pytest.mark.parametrize("K", [77, 76])  # 76: Philox players share counter blocks four at a time
def test_leapfrog_ragged_jump_and_segments(shv, orc, g, K):
    gen, seed = GENS[g]
    p = Players(shv, gen, seed, K, 5, 70)
    try:
        same(p.gen_(37), p.ref(orc, 37, offset=0))            # ragged rows: scalar path
        shv.shv_jump(p.h, shv.SHV_JUMP_DRAWS, 1003)
        p.offset += 1003
        shv.shv_set_launch_config(p.h, 1, 64, 8)              # many short segments (bits of j)
        ref = p.ref(orc, 4096)                                # (reference before the offset moves)
        same(p.gen_(4096), ref)
        shv.shv_set_launch_config(p.h, 0, 0, 0)
        ref = p.ref(orc, 1000, "f64")
        same(p.gen_(1000, "f64"), ref)
        ref = p.ref(orc, 64)
        same(p.gen_(64, host=True), ref)                      # host output path
        assert shv.shv_get_position(p.h)["players"] == K
        with pytest.raises(shv.ShvError) as ei:
            shv.shv_jump(p.h, shv.SHV_JUMP_SUBSTREAMS, 1)
        assert ei.value.status == shv.SHV_ERR_UNSUPPORTED
        with pytest.raises(shv.ShvError) as ei:
            shv.shv_get_device_view(p.h)
        assert ei.value.status == shv.SHV_ERR_UNSUPPORTED
    finally:
        p.close()


@pytest.mark.parametrize("g", list(GENS))
@pytest.mark.parametrize("K,first,n,samples", [(8, 0, 8, 5000), (4096, 100, 1000, 1001),
                                              (77, 5, 60, 3001)])  # K % 4 != 0: per-player MC kernel
def test_leapfrog_mc_matches_oracle(shv, orc, g, K, first, n, samples):
    gen, seed = GENS[g]
    p = Players(shv, gen, seed, K, first, n)
    try:
        for off in (0, 3):
            if off:
                shv.shv_jump(p.h, shv.SHV_JUMP_DRAWS, off)
            hits = torch.zeros(1, dtype=torch.int64, device="cuda")
            counts = torch.zeros(n, dtype=torch.int64, device="cuda")
            shv.shv_mc_pi_ex(p.h, samples, hits, counts, None)
            tot, ref = orc.mc_count(gen, seed, n, samples, first=first, spacing=L, players=K,
                                    offset=off + (0 if off == 0 else 2 * samples))
            assert np.array_equal(counts.cpu().numpy().view(np.uint64), ref)
            assert int(hits.item()) == tot
    finally:
        p.close()


@pytest.mark.parametrize("g", list(GENS))
def test_leapfrog_reinterleaves_base_stream_at_scale(shv, g):
    # S L418 at a size the oracle would take minutes on: 4096 players x 1024
    # draws re-interleaved equal 2^22 draws of the handle's own base stream
    # (stream 0, STREAM spacing), both from the GPU.
    gen, seed = GENS[g]
    K, m = 4096, 1024
    p = Players(shv, gen, seed, K, 0, K)
    st = torch.empty(6, dtype=torch.int32, device="cuda") if gen == W.MRG32K3A else None
    hb = shv.shv_streams_create_ex(gen, seed, 0, 1, 0, st, 0, torch.cuda.current_device(), None)
    try:
        lf = p.gen_(m)
        base = torch.empty(K * m, dtype=torch.int32, device="cuda")
        shv.shv_generate_u32(hb, base, K * m, None)
        torch.cuda.synchronize()
        assert np.array_equal(lf.T.reshape(-1), base.cpu().numpy().view(np.uint32))
    finally:
        p.close()
        shv.shv_streams_destroy(hb)


@pytest.mark.parametrize("g", list(GENS))
def test_leapfrog_c5_shape_sampled(shv, orc, g):
    # 2^20 players x 4096 u32 (16 GiB is the bench shape; 2^20 x 1024 here),
    # sampled rows against the oracle, in the default launch configuration.
    gen, seed = GENS[g]
    K, m = 1 << 20, 1024
    p = Players(shv, gen, seed, K, 0, K)
    try:
        out = p.gen_(m)
        rows = W.sample_streams(K, 48, seed=7)
        same(out[rows], p.ref(orc, m, streams=rows, offset=0))
    finally:
        p.close()


def test_leapfrog_errors(shv):
    dev = torch.cuda.current_device()
    E = shv.ShvError
    for args, code in (((W.TINYMT32, [1], 4, 0, 4), shv.SHV_ERR_MISSING_PARAMETERS),  # R19: 4 words
                       ((W.MTGP32, [1], 4, 0, 4), shv.SHV_ERR_UNSUPPORTED),
                       ((W.PHILOX4X32_10, [1], 0, 0, 4), shv.SHV_ERR_INVALID_ARGUMENT),
                       ((W.PHILOX4X32_10, [1], 4, 2, 3), shv.SHV_ERR_INSUFFICIENT_STREAMS),
                       ((W.MRG32K3A, [0] * 6, 4, 0, 4), shv.SHV_ERR_INVALID_SEED)):
        with pytest.raises(E) as ei:
            shv.shv_streams_create_leapfrog(*args, None, 0, dev, None)
        assert ei.value.status == code, args
    # base stream exhausted: Philox holds 2^66 draws, so K * draws must fit
    h = shv.shv_streams_create_leapfrog(W.PHILOX4X32_10, [1], 1 << 60, 0, 4, None, 0, dev, None)
    try:
        # player 3's draw 64 would be base draw 3 + 64 * 2^60 >= 2^66
        out = torch.empty(4 * 65, dtype=torch.int32, device="cuda")
        with pytest.raises(E) as ei:
            shv.shv_generate_u32(h, out, 65, None)
        assert ei.value.status == shv.SHV_ERR_INVALID_ARGUMENT
        shv.shv_generate_u32(h, out, 64, None)  # last base draw 3 + 63 * 2^60 < 2^66
    finally:
        shv.shv_streams_destroy(h)


# --------------------------------------------------------------------------- TinyMT32 (R19)
TM_SEED = [1, *W.TINYMT32_CHECK_PARAMS]  # {seed, mat1, mat2, tmat}


@pytest.mark.parametrize("kind", ["u32", "f32", "f64"])
@pytest.mark.parametrize("K,first,n,m", [(1, 0, 1, 700), (3, 0, 3, 301), (65, 7, 40, 256), (66, 0, 66, 64),
                                         (1000, 17, 200, 96), ((1 << 40) + 7, (1 << 39) + 5, 32, 40)])
def test_tinymt_leapfrog_matches_oracle(shv, orc, kind, K, first, n, m):
    """Stepping skips (K <= 65) and matrix skips (K > 65), far players
    (u128 jump exponents through the device tables), two calls in a row."""
    p = Players(shv, W.TINYMT32, TM_SEED, K, first, n)
    try:
        for _ in range(2):
            ref = p.ref(orc, m, kind)
            same(p.gen_(m, kind), ref)
    finally:
        p.close()


def test_tinymt_leapfrog_jump_host_and_mc(shv, orc):
    p = Players(shv, W.TINYMT32, TM_SEED, 70, 3, 50)
    try:
        same(p.gen_(37), p.ref(orc, 37, offset=0))
        shv.shv_jump(p.h, shv.SHV_JUMP_DRAWS, 1001)
        p.offset += 1001
        shv.shv_set_launch_config(p.h, 1, 64, 8)  # short segments: per-item table jumps
        ref = p.ref(orc, 300)
        same(p.gen_(300), ref)
        shv.shv_set_launch_config(p.h, 0, 0, 0)
        ref = p.ref(orc, 64)
        same(p.gen_(64, host=True), ref)
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        counts = torch.zeros(50, dtype=torch.int64, device="cuda")
        shv.shv_mc_pi_ex(p.h, 500, hits, counts, None)
        torch.cuda.synchronize()
        tot, want = orc.mc_count(W.TINYMT32, TM_SEED, 50, 500, first=3, spacing=L, players=70, offset=p.offset)
        assert np.array_equal(counts.cpu().numpy().view(np.uint64), want)
        assert int(hits.item()) == tot
    finally:
        p.close()


def test_tinymt_leapfrog_transposed_segments_sampled(shv, orc):
    """10000 players (three 4096-player segments of the transposed fill) x 256
    u32 and f32 (TMA boxes; rows past the launch clipped): sampled rows."""
    K = 10000
    p = Players(shv, W.TINYMT32, TM_SEED, K, 0, K)
    try:
        rows = [0, 1, 127, 128, 4095, 4096, 8191, 8192, 9999] + W.sample_streams(K, 16)
        for kind in ("u32", "f32"):
            ref = p.ref(orc, 256, kind, streams=rows)
            got = p.gen_(256, kind)
            same(got[rows], ref)
    finally:
        p.close()


def test_philox_transposed_counter_wrap(shv, orc):
    """Transposed Philox fill across a wrap of the low counter word (the
    hoisted round-1 product is only valid without one): K = 4 players, offset
    2^32 - 40, so lanes t = 37.. run over block 2^32."""
    p = Players(shv, W.PHILOX4X32_10, [12345, 678], 4, 0, 4)
    try:
        shv.shv_jump(p.h, shv.SHV_JUMP_DRAWS, (1 << 32) - 40)
        p.offset += (1 << 32) - 40
        for kind in ("u32", "f32"):
            ref = p.ref(orc, 64, kind)
            same(p.gen_(64, kind), ref)
    finally:
        p.close()
