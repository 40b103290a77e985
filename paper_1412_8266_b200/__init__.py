"""B200-native ShoveRand hot path (arXiv 1412.8266): bulk reproducible PRNG streams.

Thin ctypes binding over ``libshv.so`` (C ABI in ``include/shv.h``). The
functions keep the C names; this layer only marshals arguments: pointers may be
ints or objects with ``data_ptr()`` (torch tensors), CUDA streams may be ints,
``torch.cuda.Stream`` objects or None (= torch's current stream). Every status
other than SHV_OK raises :class:`ShvError`. Every step of the path runs in the
library's sm_100a kernels; there is no CPU fallback — if the library cannot be
loaded, importing this package fails.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

SHV_OK = 0
SHV_ERR_INVALID_ARGUMENT = 1
SHV_ERR_INVALID_SEED = 2
SHV_ERR_INSUFFICIENT_STREAMS = 3
SHV_ERR_UNSUPPORTED = 4
SHV_ERR_LIFECYCLE = 5
SHV_ERR_MISALIGNED = 6
SHV_ERR_EMPTY_EXPERIMENT = 7
SHV_ERR_MISSING_PARAMETERS = 8
SHV_ERR_CUDA = 9

SHV_GEN_MRG32K3A = 1
SHV_GEN_PHILOX4X32_10 = 2
SHV_GEN_TINYMT32 = 3
SHV_GEN_THREEFRY4X64_20 = 4
SHV_GEN_MTGP32 = 5
SHV_SPACING_STREAM = 0
SHV_SPACING_SUBSTREAM = 1
SHV_SPACING_KEYED = 2
SHV_SPACING_LEAPFROG = 3
SHV_JUMP_DRAWS = 0
SHV_JUMP_SUBSTREAMS = 1
SHV_JUMP_STREAMS = 2

#: Every symbol include/shv.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "shv_state_bytes", "shv_streams_create", "shv_streams_create_ex", "shv_jump",
    "shv_generate_u32", "shv_generate_f32", "shv_generate_f64", "shv_generate_u32_host",
    "shv_mc_pi", "shv_mc_pi_ex", "shv_get_position", "shv_streams_destroy",
    "shv_status_string", "shv_last_error_message", "shv_set_launch_config",
    "shv_partition", "shv_jump_matrix", "shv_build_info", "shv_get_device_view",
    "shv_streams_create_tinymt32", "shv_streams_create_leapfrog",
    "shv_verify_disjoint_workspace_bytes", "shv_verify_disjoint", "shv_streams_create_mtgp32",
)

#: Field order of shv_disjoint_report (seven u64 words, include/shv.h).
DISJOINT_REPORT_FIELDS = ("disjoint", "windows", "colliding", "pe_a", "pos_a", "pe_b", "pos_b")


class ShvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


class shv_position(C.Structure):
    _fields_ = [("gen", C.c_uint32), ("spacing", C.c_uint32), ("seed", C.c_uint32 * 6),
                ("first_stream", C.c_uint64), ("n_streams", C.c_uint64),
                ("offset_lo", C.c_uint64), ("offset_hi", C.c_uint64), ("players", C.c_uint64)]


class shv_device_view(C.Structure):
    _fields_ = [("gen", C.c_uint32), ("spacing", C.c_uint32), ("key0", C.c_uint32),
                ("key1", C.c_uint32), ("first_stream", C.c_uint64), ("n_streams", C.c_uint64),
                ("offset_lo", C.c_uint64), ("offset_hi", C.c_uint64), ("state", C.c_void_p),
                ("jump", C.c_uint32 * 18), ("params", C.c_void_p), ("group0", C.c_uint64),
                ("group_size", C.c_uint32), ("key2", C.c_uint32), ("key3", C.c_uint32)]


LIB_PATH = _build.LIB


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    st, u64, vp, u32p = C.c_int, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint32)
    sig = {
        "shv_state_bytes": (C.c_size_t, [C.c_int, u64]),
        "shv_streams_create": (st, [C.POINTER(u64), C.c_int, u32p, C.c_size_t, u64]),
        "shv_streams_create_ex": (st, [C.POINTER(u64), C.c_int, u32p, C.c_size_t, u64, u64,
                                       C.c_int, vp, C.c_size_t, C.c_int, vp]),
        "shv_jump": (st, [u64, C.c_int, u64, vp]),
        "shv_generate_u32": (st, [u64, vp, u64, vp]),
        "shv_generate_f32": (st, [u64, vp, u64, vp]),
        "shv_generate_f64": (st, [u64, vp, u64, vp]),
        "shv_generate_u32_host": (st, [u64, vp, u64, vp]),
        "shv_mc_pi": (st, [u64, u64, vp, vp]),
        "shv_mc_pi_ex": (st, [u64, u64, vp, vp, vp]),
        "shv_get_position": (st, [u64, C.POINTER(shv_position)]),
        "shv_streams_destroy": (st, [u64]),
        "shv_status_string": (C.c_char_p, [C.c_int]),
        "shv_last_error_message": (C.c_char_p, []),
        "shv_set_launch_config": (st, [u64, C.c_uint32, C.c_uint32, u64]),
        "shv_partition": (st, [u64, C.c_int, C.c_int, C.POINTER(u64), C.POINTER(u64)]),
        "shv_jump_matrix": (st, [u64, u64, u32p]),
        "shv_build_info": (C.c_char_p, []),
        "shv_get_device_view": (st, [u64, C.POINTER(shv_device_view)]),
        "shv_streams_create_tinymt32": (st, [C.POINTER(u64), u32p, C.c_size_t, C.c_uint32, C.c_uint32,
                                             u64, u64, vp, C.c_size_t, C.c_int, vp]),
        "shv_streams_create_leapfrog": (st, [C.POINTER(u64), C.c_int, u32p, C.c_size_t, u64, u64, u64,
                                             vp, C.c_size_t, C.c_int, vp]),
        "shv_verify_disjoint_workspace_bytes": (C.c_size_t, [u64, u64]),
        "shv_streams_create_mtgp32": (st, [C.POINTER(u64), u32p, C.c_size_t, u64, u64, u64, vp, C.c_size_t,
                                           C.c_int, vp]),
        "shv_verify_disjoint": (st, [vp, u64, u64, vp, C.c_size_t, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


lib = _load()


def _check(status: int):
    if status != SHV_OK:
        msg = lib.shv_last_error_message().decode()
        raise ShvError(status, f"{lib.shv_status_string(status).decode()}: {msg}")


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _stream(s) -> int:
    if s is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    if isinstance(s, int):
        return s
    return int(s.cuda_stream)


def _seed(seed):
    words = [int(w) for w in ([seed] if isinstance(seed, int) else seed)]
    arr = (C.c_uint32 * len(words))(*words)
    return arr, len(words)


def shv_state_bytes(gen: int, n_streams: int) -> int:
    return int(lib.shv_state_bytes(gen, n_streams))


def shv_streams_create(gen: int, seed, n_streams: int) -> int:
    h = C.c_uint64(0)
    arr, nw = _seed(seed)
    _check(lib.shv_streams_create(C.byref(h), gen, arr, nw, n_streams))
    return h.value


def shv_streams_create_ex(gen: int, seed, first_stream: int, n_streams: int, spacing: int,
                          d_state=None, state_bytes: int = 0, device: int = -1, stream=None) -> int:
    h = C.c_uint64(0)
    arr, nw = _seed(seed)
    if d_state is not None and not isinstance(d_state, int) and not state_bytes:
        state_bytes = d_state.numel() * d_state.element_size()
    _check(lib.shv_streams_create_ex(C.byref(h), gen, arr, nw, first_stream, n_streams, spacing,
                                     _ptr(d_state), state_bytes, device, _stream(stream)))
    return h.value


def shv_streams_create_tinymt32(params, seed: int, group_size: int, first_stream: int,
                                n_streams: int, d_state=None, state_bytes: int = 0, device: int = -1,
                                stream=None) -> int:
    """params: sequence of (mat1, mat2, tmat) records, one per group."""
    flat = [int(w) for rec in params for w in rec]
    arr = (C.c_uint32 * max(1, len(flat)))(*flat)
    h = C.c_uint64(0)
    if d_state is not None and not isinstance(d_state, int) and not state_bytes:
        state_bytes = d_state.numel() * d_state.element_size()
    _check(lib.shv_streams_create_tinymt32(C.byref(h), arr if flat else None, len(flat) // 3, seed,
                                           group_size, first_stream, n_streams, _ptr(d_state),
                                           state_bytes, device, _stream(stream)))
    return h.value


def shv_streams_create_mtgp32(params, seed: int, first_stream: int, n_streams: int, d_state=None,
                              state_bytes: int = 0, device: int = -1, stream=None) -> int:
    """MTGP32-11213 handle (R18): ``params`` = parameter records of 36 words
    (pos, sh1, sh2, mask, tbl[16], tmp_tbl[16]); family stream g uses record g."""
    h = C.c_uint64(0)
    words = [int(w) for rec in params for w in rec]
    arr = (C.c_uint32 * max(len(words), 1))(*words)
    if d_state is not None and not isinstance(d_state, int) and not state_bytes:
        state_bytes = d_state.numel() * d_state.element_size()
    _check(lib.shv_streams_create_mtgp32(C.byref(h), arr if words else None, len(words) // 36, seed,
                                         first_stream, n_streams, _ptr(d_state), state_bytes, device,
                                         _stream(stream)))
    return h.value


def shv_streams_create_leapfrog(gen: int, seed, players: int, first_player: int, n_players: int,
                                d_state=None, state_bytes: int = 0, device: int = -1,
                                stream=None) -> int:
    """Leap Frog handle: row i is player first_player + i of ``players`` (R17)."""
    h = C.c_uint64(0)
    arr, nw = _seed(seed)
    if d_state is not None and not isinstance(d_state, int) and not state_bytes:
        state_bytes = d_state.numel() * d_state.element_size()
    _check(lib.shv_streams_create_leapfrog(C.byref(h), gen, arr, nw, players, first_player, n_players,
                                           _ptr(d_state), state_bytes, device, _stream(stream)))
    return h.value


def shv_jump(h: int, kind: int, n: int, stream=None):
    _check(lib.shv_jump(h, kind, n, _stream(stream)))


def shv_generate_u32(h: int, d_out, n_per_stream: int, stream=None):
    _check(lib.shv_generate_u32(h, _ptr(d_out), n_per_stream, _stream(stream)))


def shv_generate_f32(h: int, d_out, n_per_stream: int, stream=None):
    _check(lib.shv_generate_f32(h, _ptr(d_out), n_per_stream, _stream(stream)))


def shv_generate_f64(h: int, d_out, n_per_stream: int, stream=None):
    _check(lib.shv_generate_f64(h, _ptr(d_out), n_per_stream, _stream(stream)))


def shv_generate_u32_host(h: int, h_out, n_per_stream: int, stream=None):
    _check(lib.shv_generate_u32_host(h, _ptr(h_out), n_per_stream, _stream(stream)))


def shv_mc_pi(h: int, samples_per_stream: int, d_hits, stream=None):
    _check(lib.shv_mc_pi(h, samples_per_stream, _ptr(d_hits), _stream(stream)))


def shv_mc_pi_ex(h: int, samples_per_stream: int, d_hits, d_stream_counts=None, stream=None):
    _check(lib.shv_mc_pi_ex(h, samples_per_stream, _ptr(d_hits), _ptr(d_stream_counts),
                            _stream(stream)))


def shv_get_position(h: int) -> dict:
    p = shv_position()
    _check(lib.shv_get_position(h, C.byref(p)))
    return {"gen": p.gen, "spacing": p.spacing, "seed": list(p.seed),
            "first_stream": p.first_stream, "n_streams": p.n_streams,
            "offset": p.offset_lo | (p.offset_hi << 64), "players": p.players}


def shv_get_device_view(h: int) -> shv_device_view:
    """The POD view a user kernel takes by value (include/shv_rng.cuh)."""
    v = shv_device_view()
    _check(lib.shv_get_device_view(h, C.byref(v)))
    return v


def shv_streams_destroy(h: int):
    _check(lib.shv_streams_destroy(h))


def shv_set_launch_config(h: int, blocks_per_sm: int = 0, threads_per_block: int = 0,
                          segment: int = 0):
    _check(lib.shv_set_launch_config(h, blocks_per_sm, threads_per_block, segment))


def shv_partition(total_streams: int, rank: int, world: int):
    f, c = C.c_uint64(0), C.c_uint64(0)
    _check(lib.shv_partition(total_streams, rank, world, C.byref(f), C.byref(c)))
    return f.value, c.value


def shv_jump_matrix(e: int):
    out = (C.c_uint32 * 18)()
    _check(lib.shv_jump_matrix(e & ((1 << 64) - 1), e >> 64, out))
    v = list(out)
    return [v[0:3], v[3:6], v[6:9]], [v[9:12], v[12:15], v[15:18]]


def shv_verify_disjoint_workspace_bytes(n_pe: int, horizon: int) -> int:
    return int(lib.shv_verify_disjoint_workspace_bytes(n_pe, horizon))


def shv_verify_disjoint(d_rows, n_pe: int, horizon: int, d_workspace, workspace_bytes: int,
                        d_report, stream=None):
    """Stream-ordered; d_report (7 u64 on the device, DISJOINT_REPORT_FIELDS
    order) is valid after the stream completes."""
    _check(lib.shv_verify_disjoint(_ptr(d_rows), n_pe, horizon, _ptr(d_workspace), workspace_bytes,
                                   _ptr(d_report), _stream(stream)))


def shv_status_string(s: int) -> str:
    return lib.shv_status_string(s).decode()


def shv_build_info() -> str:
    return lib.shv_build_info().decode()
