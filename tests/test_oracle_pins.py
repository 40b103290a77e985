"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Every check compares the oracle with something it does not share code with:
published constants and known-answer vectors (tests/golden/, each cited),
NVIDIA cuRAND's header implementation compiled as host code (tests/pins/),
closed forms, and invariants the generators' mathematics fixes (SPEC.md
L600-608 acceptance criteria #1, #2, #3, #7). A plausible transcription error
anywhere in the oracle (a constant, the state order, the matrix orientation,
the tie rule, the Philox lane order or key schedule, a conversion) fails at
least one of them.
"""
import math
import os
import random
import re
from fractions import Fraction

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
M1, M2 = 4294967087, 4294944443


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


# --------------------------------------------------------------------------- Philox

def test_philox_random123_kat(orc):
    for fam, *words in _rows("philox4x32_kat.txt"):
        rounds = int(fam.split("_")[1])
        v = [int(w, 16) for w in words]
        assert orc.philox_block(v[0:4], v[4:6], rounds) == v[6:10], fam


def test_philox_cpp26_required_value(orc):
    seed, nth, val = (int(x) for x in _rows("cpp26_philox4x32.txt")[0])
    # through the block function: draw nth-1 = lane 3 of block 2499
    d = nth - 1
    assert orc.philox_block([d >> 2, 0, 0, 0], [seed, 0], 10)[d & 3] == val
    # and through the stream layout (R6): stream 0, offset nth-1
    row = orc.generate(W.PHILOX4X32_10, [seed], 1, 1, offset=d)
    assert int(row[0, 0]) == val


def test_philox_block_vs_curand(orc, curand_pin):
    rng = random.Random(11)
    for _ in range(300):
        c = [rng.getrandbits(32) for _ in range(4)]
        k = [rng.getrandbits(32) for _ in range(2)]
        assert orc.philox_block(c, k, 10) == curand_pin.ask("philox", *c, *k)


@pytest.mark.parametrize("offset", [0, 1, 2, 3, 4, 5, 1001, (1 << 33) + 3, (1 << 64) - 3])
def test_philox_stream_layout_vs_curand(orc, curand_pin, offset):
    # curand_init(seed, subsequence=g, offset) + curand() serves lanes x,y,z,w
    # of ctr=(blk_lo, blk_hi, g_lo, g_hi), key=(seed_lo, seed_hi): R6.
    rng = random.Random(offset)
    for _ in range(4):
        seed = rng.getrandbits(64)
        g = rng.getrandbits(64)
        got = orc.generate(W.PHILOX4X32_10, [seed & 0xFFFFFFFF, seed >> 32], 1, 37,
                           first=g, offset=offset)[0]
        assert [int(x) for x in got] == curand_pin.ask("pstream", seed, g, offset, 37)


@pytest.mark.parametrize("offset", [0, 1, 6, 1 << 40])
def test_philox_keyed_mode_vs_curand(orc, curand_pin, offset):
    # Key-per-stream Parameterization (P L331-334, S L249-257): stream id -> key0,
    # tag -> key1, counter (blk, 0): cuRAND curand_init(tag<<32 | id, 0, offset).
    tag = 0xC0FFEE
    got = orc.generate(W.PHILOX4X32_10, [tag], 5, 29, first=77, spacing=W.SPACING_KEYED,
                       offset=offset)
    for r in range(5):
        assert [int(x) for x in got[r]] == curand_pin.ask("pstream", (tag << 32) | (77 + r), 0,
                                                           offset, 29)
    with pytest.raises(ValueError):  # key space exhausted (S L253)
        orc.generate(W.PHILOX4X32_10, [tag], 2, 4, first=(1 << 32) - 1, spacing=W.SPACING_KEYED)


def test_philox_bijective_no_collisions(orc):
    # S L230: distinct counters under one key -> no collisions over 10^6 blocks.
    rows = orc.generate(W.PHILOX4X32_10, [7, 9], 1, 4 * 1_000_000)
    blocks = rows.reshape(-1, 4).view(np.dtype((np.void, 16))).ravel()
    assert len(np.unique(blocks)) == 1_000_000


# --------------------------------------------------------------------------- MRG32k3a

def test_mrg_first_outputs_seed12345(orc):
    g = {r[0]: r[1:] for r in _rows("mrg32k3a_seed12345.txt")}
    s = [12345] * 6
    zs = []
    for _ in range(10):
        z, s = orc.mrg_step(s)
        zs.append(z)
    assert zs == [int(v) for v in g["z"]]
    assert orc.mrg_to_f64(zs[0]) == float(g["u0"][0])
    for name in ("stream1", "stream2", "stream3", "substream1", "substream2", "substream3"):
        k = int(name[-1])
        start = orc.mrg_position([12345] * 6, k if name.startswith("stream") else 0,
                                 k if name.startswith("sub") else 0, 0)
        assert start == [int(v) for v in g[name][:6]], name
        assert orc.mrg_step(start)[0] == int(g[name][6]), name


def _valid_seed(rng):
    while True:
        s = [rng.randrange(M1) for _ in range(3)] + [rng.randrange(M2) for _ in range(3)]
        if any(s[:3]) and any(s[3:]):
            return s


def test_mrg_step_vs_curand(orc, curand_pin):
    rng = random.Random(5)
    seeds = [[12345] * 6, [M1 - 1] * 3 + [M2 - 1] * 3, [1, 0, 0, 1, 0, 0], [0, 0, 1, 0, 0, 1]]
    seeds += [_valid_seed(rng) for _ in range(40)]
    for s in seeds:
        ref = curand_pin.ask("mrg", *s, 500)
        got = []
        st = list(s)
        for _ in range(500):
            z, st = orc.mrg_step(st)
            got.append(z)
        assert got == ref, s


def test_mrg_tie_maps_to_m1(orc, curand_pin):
    # R2: p1 == p2 gives z = m1 (L'Ecuyer, cuRAND), not 0.
    tie = [0, 1, 0, 0, 0, 1226359468]
    assert orc.mrg_step(tie)[0] == M1
    assert curand_pin.ask("mrg", *tie, 1) == [M1]
    # R11: SPEC L137's example state does NOT produce 0.
    assert orc.mrg_step([0, 0, 1, 0, 0, 1])[0] == 4294439475
    assert curand_pin.ask("mrg", 0, 0, 1, 0, 0, 1, 1) == [4294439475]


def test_jump_matrices_vs_rngstreams(orc):
    A1, A2 = orc.mrg_matrices()
    g = {r[0]: [int(v) for v in r[1:]] for r in _rows("rngstream_matrices.txt")}
    flat = lambda M: [v for row in M for v in row]
    assert flat(orc.mat_pow(A1, 1 << 76, M1)) == g["A1p76"]
    assert flat(orc.mat_pow(A2, 1 << 76, M2)) == g["A2p76"]
    assert flat(orc.mat_pow(A1, 1 << 127, M1)) == g["A1p127"]
    assert flat(orc.mat_pow(A2, 1 << 127, M2)) == g["A2p127"]


def _curand_tables():
    path = "/usr/local/cuda/include/curand_mrg32k3a.h"
    if not os.path.exists(path):
        pytest.skip("cuRAND headers not present")
    txt = open(path).read()
    out = {}
    for name in ("mrg32k3aM1", "mrg32k3aM2", "mrg32k3aM1SubSeq", "mrg32k3aM2SubSeq",
                 "mrg32k3aM1Seq", "mrg32k3aM2Seq"):
        m = re.search(r"unsigned int %s\[(\d+)\]\[3\]\[3\] = \{(.*?)\};" % name, txt, re.S)
        nums = [int(v) for v in re.findall(r"(\d+)u", m.group(2))]
        out[name] = np.array(nums, dtype=np.uint64).reshape(-1, 3, 3)  # SubSeq: 51 of [56] filled
    return out


def test_jump_matrices_vs_curand_tables(orc):
    # cuRAND precalc: M[i] = A^(2^i), SubSeq[i] = A^(2^(76+i)), Seq[i] = A^(2^(127+i)).
    t = _curand_tables()
    A1, A2 = orc.mrg_matrices()
    for comp, A, m in (("1", A1, M1), ("2", A2, M2)):
        for i in range(64):
            assert orc.mat_pow(A, 1 << i, m) == t["mrg32k3aM%s" % comp][i].tolist()
        for i in range(51):
            assert orc.mat_pow(A, 1 << (76 + i), m) == t["mrg32k3aM%sSubSeq" % comp][i].tolist()
        S127 = orc.mat_pow(A, 1 << 127, m)  # exponents beyond 2^128: chain the powers
        for i in range(64):
            assert orc.mat_pow(S127, 1 << i, m) == t["mrg32k3aM%sSeq" % comp][i].tolist()


def test_position_vs_curand_skipahead(orc, curand_pin):
    rng = random.Random(3)
    for _ in range(40):
        s = _valid_seed(rng)
        g = rng.getrandbits(rng.choice([1, 8, 40, 64]))
        u = rng.getrandbits(rng.choice([1, 10, 51]))
        o = rng.getrandbits(rng.choice([1, 20, 64]))
        assert orc.mrg_position(s, g, u, o) == curand_pin.ask("mrgskip", *s, g, u, o)


def test_jump_equals_iterate(orc):
    # SPEC L600 acceptance #1: 100 random n in [0, 10^6].
    rng = random.Random(1)
    seed = _valid_seed(rng)
    base = orc.generate(W.MRG32K3A, seed, 1, 1_000_008)[0]
    for n in [0, 1, 2, 3, 7, 100, 2000, 123456] + [rng.randrange(1_000_001) for _ in range(100)]:
        got = orc.generate(W.MRG32K3A, seed, 1, 8, offset=n)[0]
        assert np.array_equal(got, base[n:n + 8]), n
    # and state-level: jump(n) == n steps (SPEC L165 example n = 123456)
    s = list(seed)
    for _ in range(123456):
        _, s = orc.mrg_step(s)
    assert orc.mrg_jump(seed, 123456) == s


def test_jump_homomorphism_120bit(orc):
    # SPEC L601 acceptance #2: J(a) J(b) = J(a+b) for random 120-bit a, b.
    rng = random.Random(2)
    A1, A2 = orc.mrg_matrices()
    for _ in range(100):
        a, b = rng.getrandbits(120), rng.getrandbits(120)
        for A, m in ((A1, M1), (A2, M2)):
            assert orc.mat_mul(orc.mat_pow(A, a, m), orc.mat_pow(A, b, m), m) == \
                orc.mat_pow(A, a + b, m)


def test_stream_geometry(orc):
    # P L264-268: 2^64 streams x 2^127 = 2^191; 2^127 / 2^76 = 2^51 substreams.
    A1, A2 = orc.mrg_matrices()
    for A, m in ((A1, M1), (A2, M2)):
        assert orc.mat_pow(orc.mat_pow(A, 1 << 76, m), 1 << 51, m) == orc.mat_pow(A, 1 << 127, m)
        # full period 2^191 - 1 ... the component periods divide m^3 - 1: A^(m^3-1) = I
        assert orc.mat_pow(A, m ** 3 - 1, m) == [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
    # substream adjacency (S L173)
    s = [12345] * 6
    assert orc.mrg_jump(orc.mrg_position(s, 0, 1, 0), 1 << 76) == orc.mrg_position(s, 0, 2, 0)
    assert orc.mrg_position(s, 3, 0, 0) == orc.mrg_position(s, 2, 1 << 51, 0)


def test_oracle_rejects_invalid_seeds(orc):
    for bad in ([0] * 6, [1, 1, 1, 0, 0, 0], [M1, 1, 1, 1, 1, 1], [1, 1, 1, 1, 1, M2], [1, 2]):
        with pytest.raises(ValueError):
            orc.generate(W.MRG32K3A, bad, 1, 1)
    with pytest.raises(ValueError):
        orc.generate(W.PHILOX4X32_10, [1, 2, 3], 1, 1)
    with pytest.raises(ValueError):
        orc.generate(W.PHILOX4X32_10, [1], 1, 1, spacing=W.SPACING_SUBSTREAM)


# --------------------------------------------------------------------------- conversions

def test_norm_constant_and_f64_range(orc):
    # R7: L'Ecuyer's norm as binary64; u = fl(z * norm) in (0, 1) for z in [1, m1].
    assert float.hex(orc.mrg_to_f64(1)) == "0x1.000000d00000bp-32"
    assert 0.0 < orc.mrg_to_f64(1) and orc.mrg_to_f64(M1) < 1.0
    rng = random.Random(4)
    norm = float.fromhex("0x1.000000d00000bp-32")
    for z in [1, 2, M1 - 1, M1] + [rng.randrange(1, M1 + 1) for _ in range(2000)]:
        # one correctly-rounded multiply: compare with exact rational rounding
        exact = Fraction(z) * Fraction(norm)
        got = orc.mrg_to_f64(z)
        assert abs(Fraction(got) - exact) <= Fraction(math.ulp(got)) / 2


def test_f32_and_philox_f64_exact(orc):
    rng = random.Random(6)
    for w in [0, 1, 255, 256, 0xFFFFFFFF] + [rng.getrandbits(32) for _ in range(2000)]:
        assert Fraction(orc.to_f32(w)) == Fraction(w >> 8, 1 << 24)
    for _ in range(2000):
        lo, hi = rng.getrandbits(32), rng.getrandbits(32)
        assert Fraction(orc.philox_to_f64(lo, hi)) == Fraction(((hi << 32) | lo) >> 11, 1 << 53)
    assert orc.philox_to_f64(0xFFFFFFFF, 0xFFFFFFFF) < 1.0
    assert orc.to_f32(0xFFFFFFFF) < 1.0


def test_rows_ranges_and_conversions_agree(orc):
    for gen, sp in ((W.MRG32K3A, 1), (W.PHILOX4X32_10, 0)):
        u = orc.generate(gen, [12345], 16, 512, spacing=sp).astype(np.uint64)
        f = orc.generate(gen, [12345], 16, 512, spacing=sp, kind=orc.F32)
        assert np.array_equal(f, (u >> 8).astype(np.float32) * np.float32(2.0 ** -24))
        d = orc.generate(gen, [12345], 16, 256, spacing=sp, kind=orc.F64)
        if gen == W.MRG32K3A:
            assert u.min() >= 1 and u.max() <= M1
            norm = float.fromhex("0x1.000000d00000bp-32")
            assert np.array_equal(d, u[:, :256].astype(np.float64) * norm)
        else:
            lo, hi = u[:, 0::2], u[:, 1::2]
            ref = ((hi << np.uint64(32)) | lo) >> np.uint64(11)
            assert np.array_equal(d, ref.astype(np.float64) * 2.0 ** -53)
        assert d.min() > 0.0 if gen == W.MRG32K3A else d.min() >= 0.0
        assert d.max() < 1.0


# --------------------------------------------------------------------------- layout / replay

@pytest.mark.parametrize("gen,sp", [(W.MRG32K3A, 0), (W.MRG32K3A, 1), (W.PHILOX4X32_10, 0)])
def test_offset_replay_and_thread_invariance(orc, gen, sp):
    full = orc.generate(gen, [12345], 9, 300, spacing=sp, first=5, nthreads=1)
    for k in (1, 2, 3, 5, 7, 100):
        part = orc.generate(gen, [12345], 9, 300 - k, spacing=sp, first=5, offset=k, nthreads=3)
        assert np.array_equal(part, full[:, k:])
    assert np.array_equal(full, orc.generate(gen, [12345], 9, 300, spacing=sp, first=5, nthreads=7))
    lst = orc.generate(gen, [12345], 0, 300, spacing=sp, first=5, streams=[8, 0, 3])
    assert np.array_equal(lst, full[[8, 0, 3]])
    # first_stream shifts handle streams (R4)
    assert np.array_equal(orc.generate(gen, [12345], 4, 300, spacing=sp, first=10), full[5:9])


def test_philox_f64_straddles_blocks(orc):
    u = orc.generate(W.PHILOX4X32_10, [3, 4], 2, 64, offset=1).astype(np.uint64)
    d = orc.generate(W.PHILOX4X32_10, [3, 4], 2, 32, offset=1, kind=orc.F64)
    ref = ((u[:, 1::2] << np.uint64(32)) | u[:, 0::2]) >> np.uint64(11)
    assert np.array_equal(d, ref.astype(np.float64) * 2.0 ** -53)


# --------------------------------------------------------------------------- Monte Carlo

def test_lattice_hit_probability_closed_form():
    # R9: #{(X,Y) in [0,2^24)^2 : X^2+Y^2 < 2^48} = sum_X (isqrt(2^48 - X^2 - 1) + 1).
    X = np.arange(1 << 24, dtype=np.int64)
    r = (1 << 48) - X * X - 1
    y = np.sqrt(r.astype(np.float64)).astype(np.int64)
    y -= (y * y > r)
    y += ((y + 1) * (y + 1) <= r)
    count = int((y + 1).sum())
    assert count == 221069946527026  # SURVEY App. A D9 (independent scratch)
    assert abs(4 * count / 2 ** 48 - math.pi) < 3e-7


@pytest.mark.parametrize("gen,sp", [(W.MRG32K3A, 1), (W.PHILOX4X32_10, 0)])
def test_mc_count_recount_from_rows(orc, gen, sp):
    # sample k uses draws 2k, 2k+1 from the offset (R9); recount from the rows.
    for off in (0, 1, 3):
        tot, counts = orc.mc_count(gen, [12345], 16, 1000, spacing=sp, first=2, offset=off)
        u = orc.generate(gen, [12345], 16, 2000, spacing=sp, first=2, offset=off).astype(np.uint64)
        X, Y = u[:, 0::2] >> np.uint64(8), u[:, 1::2] >> np.uint64(8)
        ref = ((X * X + Y * Y) < np.uint64(1 << 48)).sum(axis=1)
        assert np.array_equal(counts, ref) and tot == int(ref.sum())


def test_mc_pi_within_4_sigma(orc):
    p = 221069946527026 / 2 ** 48
    for gen, sp in ((W.MRG32K3A, 1), (W.PHILOX4X32_10, 0)):
        N = 256 * (1 << 14)
        tot, _ = orc.mc_count(gen, [12345], 256, 1 << 14, spacing=sp)
        sigma = 4 * math.sqrt(p * (1 - p) / N)
        assert abs(4 * tot / N - math.pi) <= 4 * sigma


def test_mc_survey_cross_check_first_64(orc):
    # SURVEY App. A.6 (independent scratch implementation): MRG32k3a substreams
    # 0..63 of seed 12345, 2^18 samples each -> 13179528 hits.
    tot, _ = orc.mc_count(W.MRG32K3A, [12345], 64, 1 << 18, spacing=W.SPACING_SUBSTREAM)
    assert tot == 13179528


# --------------------------------------------------------------------------- TinyMT32 (NEXT-3)

def _tm_seed(seed, gs, params):
    return W.tinymt32_seed_words(seed, gs, params)


def test_tinymt32_check_output(orc):
    rows = _rows("tinymt32_check.txt")
    m1, m2, tm, seed, *outs = rows[0]
    params = [(int(m1, 16), int(m2, 16), int(tm, 16))]
    got = orc.generate(W.TINYMT32, _tm_seed(int(seed), 1, params), 1, 10)[0]
    assert [int(x) for x in got] == [int(v) for v in outs]


def test_tinymt32_jump_equals_iterate_and_slices(orc):
    params = W.tinymt32_test_params(3)
    sd = _tm_seed(99, 4, params)
    base = orc.generate(W.TINYMT32, sd, 1, 5000, first=5)[0]
    for k in (1, 2, 3, 127, 128, 129, 1000, 4321):  # GF(2) matrix jump == k steps
        assert np.array_equal(orc.generate(W.TINYMT32, sd, 1, 16, first=5, offset=k)[0], base[k:k + 16]), k
    # slice contiguity (S L345-353): slice s advanced 2^64 draws is slice s+1
    for s in (0, 1, 2):
        a = orc.generate(W.TINYMT32, sd, 1, 32, first=4 + s, offset=1 << 64)[0]
        b = orc.generate(W.TINYMT32, sd, 1, 32, first=4 + s + 1)[0]
        assert np.array_equal(a, b), s
    # group 1 and group 2 differ (one parameter set per group, P L309-313)
    assert not np.array_equal(orc.generate(W.TINYMT32, sd, 1, 32, first=4)[0],
                              orc.generate(W.TINYMT32, sd, 1, 32, first=8)[0])
    # large jumps compose: offset X+5 equals offset X then 5 steps
    X = (1 << 70) + 12340
    a = orc.generate(W.TINYMT32, sd, 1, 8, first=6, offset=X + 5)[0]
    b = orc.generate(W.TINYMT32, sd, 1, 13, first=6, offset=X)[0]
    assert np.array_equal(a, b[5:13])


def test_tinymt32_rejects(orc):
    params = W.tinymt32_test_params(2)
    with pytest.raises(ValueError):  # group 2 has no parameter set
        orc.generate(W.TINYMT32, _tm_seed(1, 4, params), 1, 4, first=8)


# --------------------------------------------------------------------------- Threefry4x64-20 (NEXT-2)

_TF_R = [(14, 16), (52, 57), (23, 40), (5, 37), (25, 33), (46, 12), (58, 22), (32, 32)]
_M64 = (1 << 64) - 1


def _tf_decrypt(y, key, rounds=20):
    """Inverse of Threefry4x64 written from the round definition (SPEC S L233,
    acceptance #3: inverse-round recovery); shares nothing with the oracle."""
    ks = list(key) + [0x1BD11BDAA9FC1A22 ^ key[0] ^ key[1] ^ key[2] ^ key[3]]
    x = list(y)
    ror = lambda v, r: ((v >> r) | (v << (64 - r))) & _M64
    for r in reversed(range(rounds)):
        if r % 4 == 3:
            s = (r + 1) // 4
            x[3] = (x[3] - s) & _M64
            for i in range(4):
                x[i] = (x[i] - ks[(s + i) % 5]) & _M64
        a, b = _TF_R[r % 8]
        if r % 2 == 0:
            x[3] = ror(x[3] ^ x[2], b); x[2] = (x[2] - x[3]) & _M64
            x[1] = ror(x[1] ^ x[0], a); x[0] = (x[0] - x[1]) & _M64
        else:
            x[1] = ror(x[1] ^ x[2], b); x[2] = (x[2] - x[1]) & _M64
            x[3] = ror(x[3] ^ x[0], a); x[0] = (x[0] - x[3]) & _M64
    return [(x[i] - ks[i]) & _M64 for i in range(4)]


def test_threefry_random123_kat(orc):
    for fam, *words in _rows("threefry4x64_kat.txt"):
        rounds = int(fam.split("_")[1])
        v = [int(w, 16) for w in words]
        assert orc.threefry4x64_block(v[0:4], v[4:8], rounds) == v[8:12], fam


def test_threefry_inverse_recovers_counter(orc):
    rng = random.Random(77)
    for _ in range(1000):
        c = [rng.getrandbits(64) for _ in range(4)]
        k = [rng.getrandbits(64) for _ in range(4)]
        assert _tf_decrypt(orc.threefry4x64_block(c, k, 20), k) == c


@pytest.mark.parametrize("offset", [0, 1, 5, 8, 13, (1 << 40) + 3])
def test_threefry_stream_layout(orc, offset):
    # R16: key (s0|s1<<32, s2|s3<<32, 0, 0); ctr (blk, g, 0, 0); words lo, hi of lanes 0..3
    seed = [0x01234567, 0x89ABCDEF, 0xDEADBEEF]
    key = [seed[0] | (seed[1] << 32), seed[2], 0, 0]
    g = 1234567
    row = orc.generate(W.THREEFRY4X64_20, seed, 1, 40, first=g, offset=offset)[0]
    for j in range(40):
        d = offset + j
        out = orc.threefry4x64_block([d >> 3, g, 0, 0], key, 20)
        lane = out[(d & 7) >> 1]
        assert int(row[j]) == ((lane >> 32) if d & 1 else lane & 0xFFFFFFFF)
    full = orc.generate(W.THREEFRY4X64_20, seed, 3, 64, first=g)
    assert np.array_equal(orc.generate(W.THREEFRY4X64_20, seed, 3, 59, first=g, offset=5), full[:, 5:])


# --------------------------------------------------------------------------- Leap Frog (NEXT-4, R17)
# P L118-122 [§2.3]: the base sequence is "dealt" to K players like cards;
# player p receives base draws p, p+K, p+2K, ... (S L397, L404, L418).

LEAP_GENS = ((W.MRG32K3A, [12345]), (W.PHILOX4X32_10, [12345, 678]), (W.THREEFRY4X64_20, [1, 2, 3, 4]))


@pytest.mark.parametrize("gen,seed", LEAP_GENS)
def test_leapfrog_one_player_is_the_base_sequence(orc, gen, seed):
    base = orc.generate(gen, seed, 1, 300)
    lf = orc.generate(gen, seed, 1, 300, spacing=W.SPACING_LEAPFROG, players=1)
    assert np.array_equal(lf, base)  # S L404: LeapFrog{1}, PE 0 = the base sequence


@pytest.mark.parametrize("gen,seed", LEAP_GENS)
@pytest.mark.parametrize("K,offset", [(2, 0), (3, 5), (8, 1), (13, 0)])
def test_leapfrog_coverage_reinterleaves_base(orc, gen, seed, K, offset):
    # S L418: the K player sequences, re-interleaved round-robin, equal the base
    # sequence over K*horizon draws; a player offset o starts at base draw K*o.
    h = 40
    base = orc.generate(gen, seed, 1, K * (offset + h))[0]
    lf = orc.generate(gen, seed, K, h, spacing=W.SPACING_LEAPFROG, players=K, offset=offset)
    assert np.array_equal(lf.T.reshape(-1), base[K * offset:])
    # a sub-range of players (a rank's share) is the same rows
    sub = orc.generate(gen, seed, 2, h, spacing=W.SPACING_LEAPFROG, players=K, offset=offset,
                       first=K - 2)
    assert np.array_equal(sub, lf[K - 2:])


def test_leapfrog_mrg_far_players_vs_curand(orc, curand_pin):
    # Large K and offsets: player p draw t is base draw d = p + K*(o+t),
    # checked against cuRAND's skipahead (a different jump implementation).
    s = [12345] * 6
    for K, p, o in ((1 << 40, 12345, 7), (1000003, 999999, 1 << 30), (3, 2, 1 << 61)):
        row = orc.generate(W.MRG32K3A, s, 1, 3, spacing=W.SPACING_LEAPFROG, players=K, first=p,
                           offset=o)[0]
        for t in range(3):
            d = p + K * (o + t)
            st = curand_pin.ask("mrgskip", *s, 0, 0, d)
            assert int(row[t]) == curand_pin.ask("mrg", *st, 1)[0], (K, p, o, t)


def test_leapfrog_philox_far_players_vs_curand(orc, curand_pin):
    seed = 12345 | (678 << 32)
    for K, p, o in ((1 << 40, 12345, 7), (1000003, 999999, 1 << 30), (5, 4, 1 << 61)):
        row = orc.generate(W.PHILOX4X32_10, [12345, 678], 1, 3, spacing=W.SPACING_LEAPFROG,
                           players=K, first=p, offset=o)[0]
        for t in range(3):
            d = p + K * (o + t)
            assert int(row[t]) == curand_pin.ask("pstream", seed, 0, d, 1)[0], (K, p, o, t)


@pytest.mark.parametrize("gen,seed", LEAP_GENS)
def test_leapfrog_conversions_and_dartboard_use_player_draws(orc, gen, seed):
    # f64 / MC consume the player's own draws (R7, R9): Philox/Threefry f64 from
    # two consecutive player draws; MRG one; MC sample k from player draws 2k, 2k+1.
    K, h = 5, 64
    u = orc.generate(gen, seed, K, 2 * h, spacing=W.SPACING_LEAPFROG, players=K).astype(np.uint64)
    f = orc.generate(gen, seed, K, h, spacing=W.SPACING_LEAPFROG, players=K, kind=orc.F64)
    for r in range(K):
        for k in range(h):
            if gen == W.MRG32K3A:
                want = Fraction(int(u[r, k])) * Fraction(2.328306549295727688e-10)
                assert f[r, k] == float(want)
            else:
                m = ((int(u[r, 2 * k + 1]) << 32 | int(u[r, 2 * k])) >> 11)
                assert f[r, k] == m * 2.0 ** -53
    tot, counts = orc.mc_count(gen, seed, K, h, spacing=W.SPACING_LEAPFROG, players=K)
    X, Y = u[:, 0::2] >> 8, u[:, 1::2] >> 8
    want = ((X * X + Y * Y) < (1 << 48)).sum(axis=1)
    assert np.array_equal(counts, want) and tot == int(want.sum())


TM_LEAP_SEED = [1, *W.TINYMT32_CHECK_PARAMS]  # {seed, mat1, mat2, tmat} (R19)


def test_tinymt_leapfrog_one_player_is_the_base_sequence(orc):
    # the base sequence is the authors' init(params, seed) sequence: a TinyMT32
    # handle's stream 0 (group 0, slice 0) with the same parameter set and seed,
    # itself pinned to the authors' check output
    base = orc.generate(W.TINYMT32, W.tinymt32_seed_words(1, 1, [W.TINYMT32_CHECK_PARAMS]), 1, 500)
    lf = orc.generate(W.TINYMT32, TM_LEAP_SEED, 1, 500, spacing=W.SPACING_LEAPFROG, players=1)
    assert np.array_equal(lf, base)


@pytest.mark.parametrize("K,offset", [(2, 0), (3, 5), (65, 1), (66, 0), (200, 3)])
def test_tinymt_leapfrog_coverage_reinterleaves_base(orc, K, offset):
    # K <= 65 skips by stepping, K > 65 by the matrix T^(K-1): both must deal
    # the base sequence exactly (S L418)
    h = 24
    base = orc.generate(W.TINYMT32, TM_LEAP_SEED, 1, K * (offset + h), spacing=W.SPACING_LEAPFROG,
                        players=1)[0]
    lf = orc.generate(W.TINYMT32, TM_LEAP_SEED, K, h, spacing=W.SPACING_LEAPFROG, players=K, offset=offset)
    assert np.array_equal(lf.T.reshape(-1), base[K * offset:])
    sub = orc.generate(W.TINYMT32, TM_LEAP_SEED, 2, h, spacing=W.SPACING_LEAPFROG, players=K, offset=offset,
                       first=K - 2)
    assert np.array_equal(sub, lf[K - 2:])


def test_leapfrog_rejects_bad_plans(orc):
    L = W.SPACING_LEAPFROG
    with pytest.raises(ValueError):  # player id >= K
        orc.generate(W.MRG32K3A, [1] * 6, 2, 4, spacing=L, players=3, first=2)
    with pytest.raises(ValueError):  # TinyMT32 leap-frog takes exactly {seed, mat1, mat2, tmat} (R19)
        orc.generate(W.TINYMT32, [1, 1, 1, 0x8F7011EE, 0xFC78FF1F, 0x3793FDFF], 1, 4, spacing=L,
                     players=2)
    with pytest.raises(ValueError):  # Philox base stream exhausted (2^66 draws)
        orc.generate(W.PHILOX4X32_10, [1], 1, 4, spacing=L, players=1 << 40, offset=1 << 26)


# --------------------------------------------------------------------------- verify_disjoint (NEXT-4)
# S L407-415: windows of 4 consecutive draws; a collision is a window shared by
# two different PEs; the constructed overlapping plan collides at position 0.

def _brute_first_collision(rows):
    best = None
    for a in range(len(rows)):
        for b in range(a + 1, len(rows)):
            for i in range(len(rows[a]) - 3):
                for j in range(len(rows[b]) - 3):
                    if all(int(rows[a][i + k]) == int(rows[b][j + k]) for k in range(4)):
                        cand = (a, i, b, j)
                        best = cand if best is None or cand < best else best
    return best


def _brute_colliding(rows):
    # distinct window values that occur in at least two different rows
    values = {tuple(int(x) for x in r[i:i + 4]) for r in rows for i in range(len(r) - 3)}
    def holds(r, v):
        return any(tuple(int(x) for x in r[i:i + 4]) == v for i in range(len(r) - 3))
    return sum(1 for v in values if sum(holds(r, v) for r in rows) >= 2)


def test_verify_disjoint_matches_brute_force(orc):
    rng = np.random.default_rng(5)
    for trial in range(40):
        rows = [rng.integers(0, 3, size=int(rng.integers(4, 14))).astype(np.uint32) for _ in range(4)]
        got = orc.verify_disjoint(rows)
        want = _brute_first_collision(rows)
        assert got["disjoint"] == (want is None), trial
        if want is not None:
            assert (got["pe_a"], got["pos_a"], got["pe_b"], got["pos_b"]) == want, trial
        assert got["windows"] == sum(len(r) - 3 for r in rows)
        assert got["colliding"] == _brute_colliding(rows), trial


def test_verify_disjoint_spec_examples(orc):
    # deliberately overlapping plan: Philox streams [0,4) and [2,6) (S L414)
    a = orc.generate(W.PHILOX4X32_10, [7], 4, 200)
    b = orc.generate(W.PHILOX4X32_10, [7], 4, 200, first=2)
    r = orc.verify_disjoint(list(a) + list(b))
    assert not r["disjoint"] and (r["pe_a"], r["pos_a"], r["pe_b"], r["pos_b"]) == (2, 0, 4, 0)
    assert r["colliding"] == 2 * 197  # streams 2 and 3 appear twice: every window of both rows
    # shifted overlap: stream 1 at offset 17 is also in the plan
    c = orc.generate(W.PHILOX4X32_10, [7], 1, 100, first=1, offset=17)
    r = orc.verify_disjoint(list(a) + list(c))
    assert (r["pe_a"], r["pos_a"], r["pe_b"], r["pos_b"]) == (1, 17, 4, 0)
    # MRG32k3a Sequence Splitting, 8 PEs, horizon 10^5 (S L412); LeapFrog{2}, 10^4 (S L415)
    assert orc.verify_disjoint(list(orc.generate(W.MRG32K3A, [12345], 8, 100000)))["disjoint"]
    lf = orc.generate(W.MRG32K3A, [12345], 2, 10000, spacing=W.SPACING_LEAPFROG, players=2)
    assert orc.verify_disjoint(list(lf))["disjoint"]


# --------------------------------------------------------------------------- MTGP32 (NEXT-4c)
# [Saito.Matsumoto2012] via P L74-76, L133-136; R18. Pinned to cuRAND's own
# MTGP32 code compiled for the host (tests/pins/mtgp_host_pin.cpp) and, apart
# from any implementation, to the generator's GF(2) linear complexity.

def test_mtgp32_params_parse_matches_curand(mtgp_pin):
    P = W.mtgp32_params()
    assert len(P) == 200
    for p in (0, 1, 57, 123, 199):
        assert list(P[p]) == mtgp_pin.ask("params", p), p


@pytest.mark.parametrize("seed", [0, 12345, (1 << 40) + 7])
def test_mtgp32_matches_curand_host(orc, mtgp_pin, seed):
    P = W.mtgp32_params()
    n = 1500  # > 4 rings of N = 351 words
    streams = [0, 1, 57, 199]
    rows = orc.generate(W.MTGP32, W.mtgp32_seed_words(seed, P), 200, n, streams=streams)
    for r, p in enumerate(streams):
        assert rows[r].tolist() == mtgp_pin.ask("gen", p, seed, n), (seed, p)


def test_mtgp32_offset_first_and_kinds(orc):
    P = W.mtgp32_params(12)
    sw = W.mtgp32_seed_words(99, P)
    full = orc.generate(W.MTGP32, sw, 12, 900)
    # first / streams select the parameter set of family stream g
    assert (orc.generate(W.MTGP32, sw, 4, 900, first=8) == full[8:12]).all()
    # an offset is the same row, later (stepping)
    assert (orc.generate(W.MTGP32, sw, 12, 300, offset=600) == full[:, 600:]).all()
    # f32 = (w>>8)*2^-24; f64 = 53 bits of (w1<<32 | w0) (R7)
    f32 = orc.generate(W.MTGP32, sw, 12, 900, kind=orc.F32)
    assert (f32 == (full >> 8).astype(np.float64) * 2.0 ** -24).all()
    f64 = orc.generate(W.MTGP32, sw, 12, 450, kind=orc.F64)
    w = full.astype(np.uint64)
    assert (f64 == ((w[:, 1::2] << np.uint64(32) | w[:, 0::2]) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53).all()
    # a parameter set must exist for every family stream
    with pytest.raises(ValueError):
        orc.generate(W.MTGP32, sw, 13, 10)


def _linear_complexity(bits):
    """Berlekamp-Massey over GF(2) (bit lists as Python ints)."""
    c, b = 1, 1
    L, m = 0, 1
    rev = 0  # bit j = s_{n-j}
    for n, s in enumerate(bits):
        rev = (rev << 1) | s
        d = ((c & rev).bit_count()) & 1
        if d == 0:
            m += 1
        elif 2 * L <= n:
            t = c
            c ^= b << m
            L, b, m = n + 1 - L, t, 1
        else:
            c ^= b << m
            m += 1
    return L


@pytest.mark.parametrize("bit", [0, 31])
def test_mtgp32_linear_complexity_is_the_mersenne_exponent(orc, bit):
    """MTGP32-11213 is F2-linear with a primitive characteristic polynomial of
    degree 11213 (the Mersenne exponent): any output bit sequence has linear
    complexity exactly 11213. A wrong shift, mask, index or table breaks it."""
    P = W.mtgp32_params(3)
    n = 2 * 11213 + 400
    for p in (0, 2):
        row = orc.generate(W.MTGP32, W.mtgp32_seed_words(7, P), 3, n, streams=[p])[0]
        bits = [int(v >> bit) & 1 for v in row]
        assert _linear_complexity(bits) == 11213, p
