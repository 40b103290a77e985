"""CPU oracle for the ShoveRand hot path (arXiv 1412.8266) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product
(``paper_1412_8266_b200``) never imports it and shares no code with it.

This module is argument marshalling over ``liboracle.so`` (built from
``shv_oracle.c`` by :func:`build`). Every function of the C file cites the paper
passage it follows; see ``shv_oracle.h``. Parity-pin status: every function here
is pinned (tests/test_oracle_pins.py); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "shv_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

MRG32K3A = 1
PHILOX4X32_10 = 2
TINYMT32 = 3
THREEFRY4X64_20 = 4
MTGP32 = 5
SPACING_STREAM = 0
SPACING_SUBSTREAM = 1
SPACING_KEYED = 2
SPACING_LEAPFROG = 3
U32, F32, F64 = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11, -ffp-contract=off)."""
    hdr = os.path.join(HERE, "shv_oracle.h")
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(SRC), os.path.getmtime(hdr))):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                           "-pthread", "-Wall", "-Wextra", "-o", tmp, SRC])
    os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u32p, u64p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
        L.orc_mrg_step.restype = C.c_uint32
        L.orc_mrg_step.argtypes = [u32p]
        L.orc_mrg_matrices.argtypes = [u64p, u64p]
        L.orc_mat_mul.argtypes = [u64p, u64p, C.c_uint64, u64p]
        L.orc_mat_pow.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.orc_mrg_jump.argtypes = [u32p, C.c_uint64, C.c_uint64]
        L.orc_mrg_position.argtypes = [u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u32p]
        L.orc_philox_block.argtypes = [u32p, u32p, C.c_int, u32p]
        L.orc_threefry4x64_block.argtypes = [u64p, u64p, C.c_int, u64p]
        L.orc_to_f32.restype = C.c_float
        L.orc_to_f32.argtypes = [C.c_uint32]
        L.orc_mrg_to_f64.restype = C.c_double
        L.orc_mrg_to_f64.argtypes = [C.c_uint32]
        L.orc_philox_to_f64.restype = C.c_double
        L.orc_philox_to_f64.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_generate.restype = C.c_int
        L.orc_generate.argtypes = [C.c_int, u32p, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                   C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_int]
        L.orc_generate_list.restype = C.c_int
        L.orc_generate_list.argtypes = [C.c_int, u32p, C.c_int, C.c_uint64, u64p, C.c_uint64,
                                        C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                        C.c_void_p, C.c_int]
        L.orc_mc_count.restype = C.c_uint64
        L.orc_mc_count.argtypes = [C.c_int, u32p, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                   C.c_uint64, C.c_uint64, C.c_uint64, u64p, C.c_int]
        L.orc_mc_count_list.restype = C.c_uint64
        L.orc_mc_count_list.argtypes = [C.c_int, u32p, C.c_int, C.c_uint64, u64p, C.c_uint64,
                                        C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, u64p, C.c_int]
        L.orc_generate_leapfrog.restype = C.c_int
        L.orc_generate_leapfrog.argtypes = [C.c_int, u32p, C.c_int, C.c_uint64, C.c_uint64, u64p,
                                            C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                            C.c_void_p, C.c_int]
        L.orc_mc_count_leapfrog.restype = C.c_uint64
        L.orc_mc_count_leapfrog.argtypes = [C.c_int, u32p, C.c_int, C.c_uint64, C.c_uint64, u64p,
                                            C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p,
                                            C.c_int]
        _lib = L
    return _lib


def _u32(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a, a.ctypes.data_as(C.POINTER(C.c_uint32))


def _u64(a):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    return a, a.ctypes.data_as(C.POINTER(C.c_uint64))


def _split(x: int):
    assert 0 <= x < (1 << 128)
    return x & ((1 << 64) - 1), x >> 64


M1 = 4294967087
M2 = 4294944443


def mrg_step(state):
    """One MRG32k3a step; returns (z, new_state)."""
    s, p = _u32(np.array(state, dtype=np.uint32).copy())
    z = lib().orc_mrg_step(p)
    return int(z), [int(v) for v in s]


def mrg_matrices():
    a1, p1 = _u64(np.zeros(9))
    a2, p2 = _u64(np.zeros(9))
    lib().orc_mrg_matrices(p1, p2)
    return a1.reshape(3, 3).tolist(), a2.reshape(3, 3).tolist()


def mat_mul(A, B, m):
    a, pa = _u64(np.array(A, dtype=np.uint64).reshape(9))
    b, pb = _u64(np.array(B, dtype=np.uint64).reshape(9))
    c, pc = _u64(np.zeros(9))
    lib().orc_mat_mul(pa, pb, m, pc)
    return c.reshape(3, 3).tolist()


def mat_pow(A, e: int, m: int):
    a, pa = _u64(np.array(A, dtype=np.uint64).reshape(9))
    out, po = _u64(np.zeros(9))
    lo, hi = _split(e)
    lib().orc_mat_pow(pa, lo, hi, m, po)
    return out.reshape(3, 3).tolist()


def mrg_jump(state, e: int):
    s, p = _u32(np.array(state, dtype=np.uint32).copy())
    lo, hi = _split(e)
    lib().orc_mrg_jump(p, lo, hi)
    return [int(v) for v in s]


def mrg_position(seed, g: int = 0, u: int = 0, o: int = 0):
    sd, ps = _u32(np.array(seed, dtype=np.uint32))
    out, po = _u32(np.zeros(6))
    lo, hi = _split(o)
    lib().orc_mrg_position(ps, g, u, lo, hi, po)
    return [int(v) for v in out]


def philox_block(ctr, key, rounds: int = 10):
    c, pc = _u32(ctr)
    k, pk = _u32(key)
    out, po = _u32(np.zeros(4))
    lib().orc_philox_block(pc, pk, rounds, po)
    return [int(v) for v in out]


def threefry4x64_block(ctr, key, rounds: int = 20):
    c, pc = _u64(ctr)
    k, pk = _u64(key)
    out, po = _u64(np.zeros(4))
    lib().orc_threefry4x64_block(pc, pk, rounds, po)
    return [int(v) for v in out]


def to_f32(w: int) -> float:
    return lib().orc_to_f32(w)


def mrg_to_f64(z: int) -> float:
    return lib().orc_mrg_to_f64(z)


def philox_to_f64(lo: int, hi: int) -> float:
    return lib().orc_philox_to_f64(lo, hi)


_DT = {U32: np.uint32, F32: np.float32, F64: np.float64}


def generate(gen, seed, n_streams, n, *, first=0, spacing=SPACING_STREAM, offset=0,
             kind=U32, nthreads=None, streams=None, players=None):
    """Rows out[i, j] (R8). ``streams`` optionally lists handle-stream indices.
    spacing=SPACING_LEAPFROG deals one base sequence to ``players`` players;
    row i is player first + i (orc_stream_open_leapfrog)."""
    nthreads = nthreads or os.cpu_count() or 1
    sd, ps = _u32(seed)
    lo, hi = _split(offset)
    if spacing == SPACING_LEAPFROG:
        idx, pi = _u64(streams if streams is not None else [])
        rows = len(idx) if streams is not None else n_streams
        out = np.empty((rows, n), dtype=_DT[kind])
        rc = lib().orc_generate_leapfrog(gen, ps, len(sd), players, first,
                                         pi if streams is not None else None, rows, lo, hi, n,
                                         kind, out.ctypes.data, nthreads)
    elif streams is None:
        out = np.empty((n_streams, n), dtype=_DT[kind])
        rc = lib().orc_generate(gen, ps, len(sd), first, n_streams, spacing, lo, hi, n, kind,
                                out.ctypes.data, nthreads)
    else:
        idx, pi = _u64(streams)
        out = np.empty((len(idx), n), dtype=_DT[kind])
        rc = lib().orc_generate_list(gen, ps, len(sd), first, pi, len(idx), spacing, lo, hi, n,
                                     kind, out.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError("oracle rejected the arguments")
    return out


def mc_count(gen, seed, n_streams, samples, *, first=0, spacing=SPACING_STREAM, offset=0,
             nthreads=None, streams=None, players=None):
    """(total hits, per-stream counts) of the dartboard (R9)."""
    nthreads = nthreads or os.cpu_count() or 1
    sd, ps = _u32(seed)
    lo, hi = _split(offset)
    if spacing == SPACING_LEAPFROG:
        idx, pi = _u64(streams if streams is not None else [])
        rows = len(idx) if streams is not None else n_streams
        counts, pc = _u64(np.zeros(rows))
        tot = lib().orc_mc_count_leapfrog(gen, ps, len(sd), players, first,
                                          pi if streams is not None else None, rows, lo, hi,
                                          samples, pc, nthreads)
    elif streams is None:
        counts, pc = _u64(np.zeros(n_streams))
        tot = lib().orc_mc_count(gen, ps, len(sd), first, n_streams, spacing, lo, hi, samples,
                                 pc, nthreads)
    else:
        idx, pi = _u64(streams)
        counts, pc = _u64(np.zeros(len(idx)))
        tot = lib().orc_mc_count_list(gen, ps, len(sd), first, pi, len(idx), spacing, lo, hi,
                                      samples, pc, nthreads)
    if tot == (1 << 64) - 1:
        raise ValueError("oracle rejected the arguments")
    return int(tot), counts


def verify_disjoint(rows):
    """Disjointness audit by definition (S L407-415 verify_disjoint; S L425):
    ``rows`` = one array of u32 draws per PE, in PE order. Every window of 4
    consecutive draws is recorded with its (pe, pos); a collision is a window
    held by two different PEs. Returns {"disjoint", "windows", "colliding" (distinct
    window values held by >= 2 different PEs)} and, if not
    disjoint, the lexicographically smallest (pe_a, pos_a, pe_b, pos_b) with
    pe_a < pe_b over all colliding pairs. Plain dict of windows; no hashing
    shortcut, no sorting."""
    seen = {}
    windows = 0
    for pe, r in enumerate(rows):
        r = [int(x) for x in r]
        for pos in range(len(r) - 3):
            seen.setdefault(tuple(r[pos:pos + 4]), []).append((pe, pos))
            windows += 1
    best = None
    colliding = 0
    for occ in seen.values():
        if len(occ) < 2:
            continue
        if len({pe for pe, _ in occ}) > 1:
            colliding += 1
        for x in range(len(occ)):
            for y in range(x + 1, len(occ)):
                (pa, qa), (pb, qb) = occ[x], occ[y]
                if pa == pb:
                    continue
                cand = (pa, qa, pb, qb) if pa < pb else (pb, qb, pa, qa)
                if best is None or cand < best:
                    best = cand
    out = {"disjoint": best is None, "windows": windows, "colliding": colliding}
    if best is not None:
        out.update(pe_a=best[0], pos_a=best[1], pe_b=best[2], pos_b=best[3])
    return out
