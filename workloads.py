"""Seeded synthetic workloads shared by tests/ and bench.py (arXiv 1412.8266 hot path).

This module holds NO arithmetic of the method: only the workload shapes of
BASELINE.json ``configs`` (seeds, stream counts, draws per stream, spacing) and
a SplitMix64 index sampler used to pick which streams a parity test checks.
Both the oracle side and the CUDA side read their inputs from here; neither
imports the other.
"""
from __future__ import annotations

from dataclasses import dataclass

MRG32K3A = 1
PHILOX4X32_10 = 2
TINYMT32 = 3
THREEFRY4X64_20 = 4
MTGP32 = 5
SPACING_STREAM = 0
SPACING_SUBSTREAM = 1
SPACING_KEYED = 2
SPACING_LEAPFROG = 3  # Leap Frog partition (P L118-122): players dealt one base sequence


@dataclass(frozen=True)
class Workload:
    name: str
    gen: int
    seed: tuple
    n_streams: int
    n: int            # values per stream (fills) or samples per stream (MC)
    spacing: int = SPACING_STREAM
    first: int = 0


# BASELINE.json configs[0]: MRG32k3a, seed 12345, 4 streams x 1000 (STREAM spacing, R4).
C1 = Workload("C1", MRG32K3A, (12345,), 4, 1000, SPACING_STREAM)
# configs[1]: 2^16 counter-streams x 1024 u32, key (12345, 0) (R6).
C2 = Workload("C2", PHILOX4X32_10, (12345,), 1 << 16, 1024, SPACING_STREAM)
# configs[2]: 2^20 substreams x 4096 doubles (SUBSTREAM spacing, R4).
C3 = Workload("C3", MRG32K3A, (12345,), 1 << 20, 4096, SPACING_SUBSTREAM)
# configs[3]: MC pi, 2^38 samples over 2^20 streams (2^18 samples each).
C4_MRG = Workload("C4-mrg", MRG32K3A, (12345,), 1 << 20, 1 << 18, SPACING_SUBSTREAM)
C4_PHILOX = Workload("C4-philox", PHILOX4X32_10, (12345,), 1 << 20, 1 << 18, SPACING_STREAM)
# configs[4]: 16 GiB u32 per GPU = 2^20 streams x 4096 per rank, both generators.
C5_MRG = Workload("C5-mrg", MRG32K3A, (12345,), 1 << 20, 4096, SPACING_SUBSTREAM)
C5_PHILOX = Workload("C5-philox", PHILOX4X32_10, (12345,), 1 << 20, 4096, SPACING_STREAM)


def rank_slice(w: Workload, rank: int, world: int, weak: bool) -> Workload:
    """The stream range rank ``rank`` of ``world`` owns.

    weak=True: every rank gets w.n_streams streams starting at rank*n_streams
    (C5). weak=False: the w.n_streams streams are split into contiguous ranges
    (C4)."""
    if weak:
        return Workload(w.name, w.gen, w.seed, w.n_streams, w.n, w.spacing,
                        w.first + rank * w.n_streams)
    lo = w.n_streams * rank // world
    hi = w.n_streams * (rank + 1) // world
    return Workload(w.name, w.gen, w.seed, hi - lo, w.n, w.spacing, w.first + lo)


# TinyMT32 parameter set of the authors' check output (tinymt32dc check
# parameters): (mat1, mat2, tmat).
TINYMT32_CHECK_PARAMS = (0x8F7011EE, 0xFC78FF1F, 0x3793FDFF)


def tinymt32_test_params(k: int):
    """k parameter records for parity tests: the check set, then SplitMix64
    words. TEST-ONLY: the extra records are not Dynamic Creator output, so
    their periods are not certified; oracle and GPU must agree regardless."""
    out = [TINYMT32_CHECK_PARAMS]
    words = splitmix64(1412, 3 * k)
    for r in range(1, k):
        out.append(tuple(w & 0xFFFFFFFF for w in words[3 * r:3 * r + 3]))
    return out[:k]


def tinymt32_seed_words(seed: int, group_size: int, params):
    """The oracle's TinyMT32 seed vector: {seed, group_size, n_params, params...} (R15)."""
    return [seed, group_size, len(params)] + [w for rec in params for w in rec]


MTGP32_PARAM_HEADER = "curand_mtgp32dc_p_11213.h"


def mtgp32_params(k: int = 200):
    """The first k MTGP32-11213 parameter sets (the MTGP authors' Dynamic
    Creator output, 200 sets, as shipped in the CUDA toolkit's
    curand_mtgp32dc_p_11213.h), each as 36 words: pos, sh1, sh2, mask,
    tbl[16], tmp_tbl[16] (R18). Parsed from the header text; input data only."""
    import os
    import re
    roots = [os.environ.get("CUDA_HOME", ""), "/usr/local/cuda"]
    path = next((os.path.join(r, "include", MTGP32_PARAM_HEADER) for r in roots
                 if r and os.path.exists(os.path.join(r, "include", MTGP32_PARAM_HEADER))), None)
    if path is None:
        raise FileNotFoundError(MTGP32_PARAM_HEADER + " not found under CUDA_HOME or /usr/local/cuda")
    text = open(path).read()
    body = text[text.index("mtgp32dc_params_fast_11213[]"):]
    sets = []
    for rec in re.finditer(r"/\* No\.(\d+)[^*]*\*/(.*?)(?=/\* No\.|\};\s*$|\}\s*;)", body, re.S):
        nums = [int(v, 0) for v in re.findall(r"0x[0-9a-fA-F]+|\b\d+\b", rec.group(2))]
        # mexp, pos, sh1, sh2, tbl[16], tmp_tbl[16], flt_tmp_tbl[16], mask, poly_sha1[21]
        mexp, pos, sh1, sh2 = nums[:4]
        tbl, tmp_tbl, mask = nums[4:20], nums[20:36], nums[52]
        assert mexp == 11213, mexp
        sets.append(tuple([pos, sh1, sh2, mask] + tbl + tmp_tbl))
        if len(sets) == k:
            break
    return sets


def mtgp32_seed_words(seed: int, params):
    """The oracle's MTGP32 seed vector: {seed_lo, seed_hi, n_params, 36 words per set} (R18)."""
    return [seed & 0xFFFFFFFF, seed >> 32, len(params)] + [w for rec in params for w in rec]


def splitmix64(seed: int, count: int):
    """SplitMix64 outputs (Steele et al. 2014) — index sampling only."""
    out = []
    x = seed & 0xFFFFFFFFFFFFFFFF
    for _ in range(count):
        x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        out.append(z ^ (z >> 31))
    return out


def sample_streams(n_streams: int, k: int = 1024, seed: int = 2026):
    """Sorted unique stream indices: edges (0..3, 2^b-1, 2^b, last) plus k
    SplitMix64-drawn indices (SURVEY §8c parity selection)."""
    s = {0, 1, 2, 3, n_streams - 1}
    b = 4
    while (1 << b) <= n_streams:
        s.add((1 << b) - 1)
        if (1 << b) < n_streams:
            s.add(1 << b)
        b += 1
    s.update(v % n_streams for v in splitmix64(seed, k))
    return sorted(i for i in s if 0 <= i < n_streams)
