"""Exactness argument of the FP64 MRG32k3a step (include/shv_device.cuh:
mrg_c1_floor, mrg_c2_floor), checked with exact rationals.

The GPU step computes k = floor(p * inv) with one fma rounded toward -inf and
r = p - k*m. It is exact iff inv's rounding error delta keeps p*inv on the
same side of every integer as p/m. These tests pin the constants the header
uses and the bounds the argument needs; they do not run the kernels (the
GPU parity tests do)."""
import math
import os
import random
import struct
from fractions import Fraction as Fr

M1, M2 = 4294967087, 4294944443
A12, A13N, A21, A23N = 1403580, 810728, 527612, 1370589
INV1 = 1.0 / M1                       # RN(1/m1)
INV2 = float.fromhex("0x1.000059451f212p-32")  # RU(1/m2)
HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "shv_device.cuh")


def floor_red(p: int, inv: float, m: int) -> int:
    """r = p - floor(p*inv)*m with p*inv exact (the fma's exact product, then RD)."""
    return p - math.floor(Fr(p) * Fr(inv)) * m


def test_header_constants():
    src = open(HDR).read()
    assert "0x1.000059451f212p-32" in src and "1.0 / (double)kM1" in src
    assert INV2 == math.nextafter(1.0 / M2, 1.0)  # RU(1/m2): RN(1/m2) rounds down
    assert A23N * M2 == 5886603609186927 and float(A23N * M2) == A23N * M2 < 2**53


def test_inverse_errors_and_bounds():
    d1 = Fr(INV1) - Fr(1, M1)
    d2 = Fr(INV2) - Fr(1, M2)
    assert d1 > 0 and d2 > 0
    # component 1: signed form, states in [0, m1] -> |p| <= max(a12, a13n) * m1 < 2^53
    p1max = max(A12, A13N) * M1
    assert p1max < 2**53 and p1max * M1 * d1 < 1
    # component 2: positive form a21*y2 + a23n*(m2 - y0), y in [0, m2)
    p2max = A21 * (M2 - 1) + A23N * M2
    assert p2max < 2**53 and p2max * M2 * d2 < 1


def test_floor_reduction_edges_and_random():
    rng = random.Random(1412)
    # component 2: always the canonical residue
    cases = [0, 1, M2 - 1, M2, M2 + 1, A23N * M2, A21 * (M2 - 1) + A23N * M2]
    cases += [k * M2 + r for k in (1, 7, 1 << 20) for r in (0, 1, M2 - 1)]
    for _ in range(20000):
        y0, y2 = rng.randrange(M2), rng.randrange(M2)
        cases.append(A21 * y2 + A23N * (M2 - y0))
    for p in cases:
        assert floor_red(p, INV2, M2) == p % M2, p
    # component 1: canonical, or m1 when p is a negative multiple of m1
    cases = [0, 1, -1, M1 - 1, -(M1 - 1), M1, -M1, A12 * M1, -A13N * M1]
    cases += [s * (k * M1 + r) for s in (1, -1) for k in (1, 5, 1 << 19) for r in (0, 1, M1 - 1)]
    for _ in range(20000):
        x0, x1 = rng.randrange(M1 + 1), rng.randrange(M1 + 1)
        cases.append(A12 * x1 - A13N * x0)
    for p in cases:
        r = floor_red(p, INV1, M1)
        assert r == p % M1 or (r == M1 and p % M1 == 0 and p < 0), p
        assert 0 <= r <= M1


def test_combine_maps_m1_like_zero():
    # mrg_combine(p1, p2) = p1 - p2 (+ m1 if p1 <= p2), wrap-around u32
    def comb(p1, p2):
        z = (p1 - p2) % 2**32
        return (z + M1) % 2**32 if p1 <= p2 else z
    for p2 in (0, 1, 12345, M2 - 1):
        assert comb(M1, p2) == comb(0, p2)


def c1_int(x0: int, x1: int) -> int:
    """The integer half-step mrg_c1_int (include/shv_device.cuh) in u32 arithmetic,
    instruction by instruction: t = m1 - x0; P = a12*x1 + a13n*t (u64); (H, L);
    u = L + 209*H mod 2^32; p1 = u + 209 if (u < L or u >= m1) else u."""
    t = (M1 - x0) % 2**32
    P = A12 * x1 + A13N * t
    assert P < 2**64
    return fold1(P)


def fold1(P: int) -> int:
    H, L = P >> 32, P & 0xFFFFFFFF
    u = (L + 209 * H) % 2**32
    return (u + 209) % 2**32 if (u < L or u >= M1) else u


def test_integer_half_step_bounds():
    # P = a12*x1 + a13n*(m1 - x0) for canonical x < m1: its high word times 209
    # stays below 2^32, so u wraps at most once (u < L detects it)
    pmax = A12 * (M1 - 1) + A13N * M1
    assert pmax < 2**53.1 and 209 * (pmax >> 32) < 2**28.8
    rng = random.Random(8266)
    hmax = pmax >> 32
    for H in [0, 1, 2, 3, hmax - 1, hmax] + [rng.randrange(hmax + 1) for _ in range(200)]:
        c = 209 * H
        for L in {0, 1, 208, 209, (M1 - c - 1) % 2**32, (M1 - c) % 2**32, (2**32 - c - 1) % 2**32,
                  (2**32 - c) % 2**32, 2**32 - 1, M1 - 1, M1, rng.randrange(2**32)}:
            P = (H << 32) | L
            if P <= pmax:
                assert fold1(P) == P % M1, (H, L)
    for x0, x1 in [(0, 0), (0, M1 - 1), (M1 - 1, 0), (M1 - 1, M1 - 1), (1, 1), (0, 1)]:
        assert c1_int(x0, x1) == (A12 * x1 - A13N * x0) % M1
    for _ in range(50000):
        x0, x1 = rng.randrange(M1), rng.randrange(M1)
        assert c1_int(x0, x1) == (A12 * x1 - A13N * x0) % M1


# ---- MrgSN: the subnormal-state step (include/shv_device.cuh mrg_c1_sn / mrg_c2_sn)

def D(v: int) -> float:
    """The register pair {v_lo, v_hi} as a double (v < 2^64): for v < 2^53 this is
    v * 2^-1074 exactly (subnormal below 2^52, exponent field 1 above)."""
    return struct.unpack("<d", struct.pack("<Q", v))[0]


def bits(d: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", d))[0]


SN_C1Q = float.fromhex("0x0.317b9fd79a126p-1022")
SN_C2P = float.fromhex("0x1.4e9d5b50f226fp-1022")
SN_C1S = float.fromhex("0x1.000000d10000bp+980")
SN_C2S = float.fromhex("0x1.000059451f212p+978")
SN_M = float.fromhex("0x1.8p-12")


def fma_rd_lo(a: float, b: float, c: float) -> int:
    """Low word of fma.rm(a, b, c) for c = 1.5*2^-12 and 0 <= a*b < 2^-33:
    the exact a*b + c rounded down to the ulp of [2^-12, 2^-11), 2^-64."""
    v = Fr(a) * Fr(b) + Fr(c)
    q = math.floor(v * 2**64)
    assert Fr(2**-12) <= Fr(q, 2**64) < Fr(2**-11)
    return bits(float(Fr(q, 2**64))) & 0xFFFFFFFF


def c1_sn(x0: int, x1: int) -> int:
    t = -202682.0 * D(x0) + SN_C1Q      # exact: the fma's product and sum are representable
    q = 350895.0 * D(x1) + t
    assert bits(q) == 350895 * x1 + 202682 * (M1 - x0)
    k = fma_rd_lo(q, SN_C1S, SN_M)
    return (4 * (bits(q) & 0xFFFFFFFF) + 209 * k) % 2**32


def c2_sn(y0: int, y2: int) -> int:
    t = -float(A23N) * D(y0) + SN_C2P
    p = float(A21) * D(y2) + t
    assert bits(p) == A21 * y2 + A23N * (M2 - y0)
    k = fma_rd_lo(p, SN_C2S, SN_M)
    return ((bits(p) & 0xFFFFFFFF) + 22853 * k) % 2**32


def test_sn_constants():
    src = open(HDR).read()
    for h in ("0x0.317b9fd79a126p-1022", "0x1.4e9d5b50f226fp-1022", "0x1.000000d10000bp+980",
              "0x1.000059451f212p+978", "0x1.8p-12"):
        assert h in src, h
    assert bits(SN_C1Q) == 202682 * M1 and bits(SN_C2P) == A23N * M2
    assert Fr(SN_C1S) == 4 * Fr(INV1) * 2**1010 and Fr(SN_C2S) == Fr(INV2) * 2**1010
    assert SN_M == 1.5 * 2**-12
    for v in (0, 1, 2**32 - 1, 2**52 - 1, 2**52, 2**53 - 1):  # the bit pattern of D(v) is v
        assert Fr(D(v)) == Fr(v, 2**1074) and bits(D(v)) == v
    assert 4 * 350895 == A12 and 4 * 202682 == A13N


def test_sn_bounds():
    d1 = Fr(INV1) - Fr(1, M1)
    d2 = Fr(INV2) - Fr(1, M2)
    qmax = 350895 * (M1 - 1) + 202682 * M1          # x canonical: x1 <= m1 - 1, m1 - x0 <= m1
    assert qmax < 2**51.08 < 2**52 and 4 * qmax * M1 * d1 < Fr(72, 100)
    pmax = A21 * (M2 - 1) + A23N * M2
    assert pmax < 2**52.86 and pmax * M2 * d2 < Fr(98, 100)
    # the quotients fit below the ulp-2^-64 window: M + k * 2^-64 < 2^-11
    assert 4 * qmax // M1 < 2**22 and pmax // M2 < 2**22


def test_sn_step_emulated_matches_recurrence():
    rng = random.Random(14128266)
    edges1 = [0, 1, 2, M1 - 2, M1 - 1]
    edges2 = [0, 1, 2, M2 - 2, M2 - 1]
    for x0 in edges1:
        for x1 in edges1:
            assert c1_sn(x0, x1) == (A12 * x1 - A13N * x0) % M1
    for y0 in edges2:
        for y2 in edges2:
            assert c2_sn(y0, y2) == (A21 * y2 - A23N * y0) % M2
    # quotient boundaries: 4q = k m1 + {0, 1, m1 - 1}, p = k m2 + {0, 1, m2 - 1}
    i13, i23 = pow(A13N, -1, M1), pow(A23N, -1, M2)
    for _ in range(100):
        x1, y2 = rng.randrange(M1), rng.randrange(M2)
        for res in (0, 1, M1 - 1):
            x0 = (A12 * x1 - res) * i13 % M1
            assert (A12 * x1 + A13N * (M1 - x0)) % M1 == res
            assert c1_sn(x0, x1) == res
        for res in (0, 1, M2 - 1):
            y0 = (A21 * y2 - res) * i23 % M2
            assert c2_sn(y0, y2) == res
    for _ in range(300):
        x0, x1 = rng.randrange(M1), rng.randrange(M1)
        assert c1_sn(x0, x1) == (A12 * x1 - A13N * x0) % M1
        y0, y2 = rng.randrange(M2), rng.randrange(M2)
        assert c2_sn(y0, y2) == (A21 * y2 - A23N * y0) % M2
    # a run of the full step from a seed, against the recurrence
    x = [12345, 12345, 12345]
    y = [12345, 12345, 12345]
    for _ in range(2000):
        n1 = c1_sn(x[0], x[1])
        assert n1 == (A12 * x[1] - A13N * x[0]) % M1
        n2 = c2_sn(y[0], y[2])
        assert n2 == (A21 * y[2] - A23N * y[0]) % M2
        x = [x[1], x[2], n1]
        y = [y[1], y[2], n2]


def test_sn_lane_start_split_row():
    """split_row_sn (kernels_mrg.cu): Ah = sum Mh v, Al = sum Ml v with 16-bit
    halves, rh = Ah mod m by the plain inverse RN(1/m1) 2^1010 (c_mrg_snk[5]) or
    RU(1/m2) 2^1010, X = rh 2^16 + Al, r = X mod m; emulated with exact rationals."""
    src = open(os.path.join(os.path.dirname(HDR), "..", "paper_1412_8266_b200", "csrc", "kernels_mrg.cu")).read()
    assert "0x1.000000d10000bp+978" in src
    c1u = float.fromhex("0x1.000000d10000bp+978")
    assert Fr(c1u) == Fr(INV1) * 2**1010
    amax = 3 * 65535 * (2**32 - 1)
    xmax = (M1 - 1) * 2**16 + amax
    assert amax < 2**49.6 and xmax < 2**50
    for d, m in ((Fr(INV1) - Fr(1, M1), M1), (Fr(INV2) - Fr(1, M2), M2)):
        assert xmax * m * d < 1 and amax * m * d < 1
    rng = random.Random(2026)

    def row(Mrow, v, cinv, m, c):
        ah = sum((Mq >> 16) * vq for Mq, vq in zip(Mrow, v))
        al = sum((Mq & 0xFFFF) * vq for Mq, vq in zip(Mrow, v))
        rh = ((ah & 0xFFFFFFFF) + c * fma_rd_lo(D(ah), cinv, SN_M)) % 2**32
        x = rh * 65536 + al
        return ((x & 0xFFFFFFFF) + c * fma_rd_lo(D(x), cinv, SN_M)) % 2**32
    for m, c, cinv in ((M1, 209, c1u), (M2, 22853, SN_C2S)):
        for _ in range(400):
            Mrow = [rng.choice([0, 1, m - 1, rng.randrange(m)]) for _ in range(3)]
            v = [rng.choice([0, 1, m - 1, rng.randrange(m)]) for _ in range(3)]
            assert row(Mrow, v, cinv, m, c) == sum(a * b for a, b in zip(Mrow, v)) % m


# ---- MrgMF: magic-free subnormal quotients (include/shv_device.cuh, MrgMF)

def mul_rd_sub(a: float, b: float) -> float:
    """mul.rm(a, b) for a subnormal-range result (|a*b| < 2^-1022): the exact
    product rounded toward -inf onto the 2^-1074 grid (IEEE 754 directed rounding;
    every subnormal has ulp 2^-1074)."""
    v = Fr(a) * Fr(b)
    assert abs(v) < Fr(2) ** -1022
    q = math.floor(v * 2**1074)
    return float(Fr(q, 2**1074))


def c1_mf(x0: int, x1: int) -> int:
    t = 810728.0 * D(x0)                       # exact products and sums (integers < 2^53 units)
    p = 1403580.0 * D(x1) - t
    assert Fr(p) * 2**1074 == A12 * x1 - A13N * x0
    k = mul_rd_sub(p, INV1)                    # D(floor(p / m1)), sign allowed
    r = float(Fr(p) - Fr(k) * M1)              # fma(-k, m1, p): exact (r is an integer < 2^32 units)
    assert Fr(r) == Fr(p) - Fr(k) * M1
    return bits(r)                             # the pair {r, 0}: r in [0, m1]


def c2_mf(y0: int, y2: int) -> int:
    t = -float(A23N) * D(y0) + SN_C2P
    p = float(A21) * D(y2) + t
    k = mul_rd_sub(p, INV2)
    r = float(Fr(p) - Fr(k) * M2)
    return bits(r)


def test_mf_step_emulated_matches_recurrence():
    rng = random.Random(20261018)
    i13, i23 = pow(A13N, -1, M1), pow(A23N, -1, M2)
    for x0 in (0, 1, M1 - 1, M1):
        for x1 in (0, 1, M1 - 1, M1):
            r = c1_mf(x0, x1)
            assert r < 2**32 and (r == (A12 * x1 - A13N * x0) % M1 or (r == M1 and (A12 * x1 - A13N * x0) % M1 == 0))
    for _ in range(300):  # quotient boundaries: p = k m + {0, 1, m - 1}
        x1, y2 = rng.randrange(M1), rng.randrange(M2)
        for res in (0, 1, M1 - 1):
            x0 = (A12 * x1 - res) * i13 % M1
            r = c1_mf(x0, x1)
            assert r == res or (res == 0 and r == M1 and A12 * x1 - A13N * x0 < 0)
        for res in (0, 1, M2 - 1):
            y0 = (A21 * y2 - res) * i23 % M2
            assert c2_mf(y0, y2) == res
    x = [12345] * 3
    y = [12345] * 3
    for _ in range(2000):
        n1, n2 = c1_mf(x[0], x[1]), c2_mf(y[0], y[2])
        assert n1 % M1 == (A12 * x[1] - A13N * x[0]) % M1 and n1 <= M1
        assert n2 == (A21 * y[2] - A23N * y[0]) % M2
        x = [x[1], x[2], n1]
        y = [y[1], y[2], n2]
