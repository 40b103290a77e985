"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bar (R1-R12): every u32 value, and every f32/f64 value as a bit
pattern, equal to the oracle's on the same seeded workload — integer work is
bit-exact, and the conversions are exact or one correctly-rounded multiply.
Small configs are compared in full (several segments, ragged tails); the full
BASELINE.json sizes are compared on sampled streams (workloads.sample_streams)
and on whole-output checksums written by tests/golden/make_golden.py (oracle
only), in the launch configuration bench.py uses.
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = os.path.join(os.path.dirname(__file__), "golden")
M1 = 4294967087


@pytest.fixture(scope="module")
def shv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1412_8266_b200 as shv
    return shv


DT = {"u32": (torch.int32, np.uint32), "f32": (torch.float32, np.float32),
      "f64": (torch.float64, np.float64)}


class Fam:
    """A handle plus the arguments the oracle needs to replay it."""

    def __init__(self, shv, gen, seed, n_streams, spacing=0, first=0):
        self.shv, self.gen, self.seed = shv, gen, list(seed) if not isinstance(seed, int) else [seed]
        self.n_streams, self.spacing, self.first = n_streams, spacing, first
        self.state = None
        if gen == W.MRG32K3A:
            self.state = torch.empty(6 * n_streams, dtype=torch.int32, device="cuda")
        self.h = shv.shv_streams_create_ex(gen, self.seed, first, n_streams, spacing, self.state,
                                           0, torch.cuda.current_device(), None)
        self.offset = 0

    def gen_(self, n, kind="u32", out=None):
        tdt, ndt = DT[kind]
        if out is None:
            out = torch.empty(self.n_streams * n, dtype=tdt, device="cuda")
        getattr(self.shv, "shv_generate_" + kind)(self.h, out, n, None)
        torch.cuda.synchronize()
        self.offset += n * (2 if (kind == "f64" and self.gen != W.MRG32K3A) else 1)
        return out.cpu().numpy().view(ndt).reshape(self.n_streams, n) if n else out

    def ref(self, orc, n, kind="u32", offset=None, streams=None):
        return orc.generate(self.gen, self.seed, self.n_streams, n, first=self.first,
                            spacing=self.spacing, offset=self.offset if offset is None else offset,
                            kind={"u32": 0, "f32": 1, "f64": 2}[kind], streams=streams)

    def close(self):
        self.shv.shv_streams_destroy(self.h)


def same(a, b):
    assert a.shape == b.shape
    if a.dtype.kind == "f":
        a = a.view(np.uint32 if a.itemsize == 4 else np.uint64)
        b = b.view(a.dtype)
    bad = np.nonzero(a != b)
    assert len(bad[0]) == 0, f"{len(bad[0])} mismatches, first at {[x[:5] for x in bad]}"


# ---------------------------------------------------------------- C1

@pytest.mark.parametrize("kind", ["u32", "f32", "f64"])
def test_c1_mrg_4x1000_full(shv, orc, kind):
    f = Fam(shv, W.MRG32K3A, W.C1.seed, W.C1.n_streams, W.C1.spacing)
    ref = f.ref(orc, W.C1.n, kind)
    got = f.gen_(W.C1.n, kind)
    same(got, ref)
    if kind == "u32":  # SURVEY App. A.2 first/last values
        assert got[:, 0].tolist() == [545508589, 3262379099, 3128925555, 411039607]
        assert got[:, 999].tolist() == [4235174647, 1962922018, 1313695736, 2457220498]
    f.close()


# ---------------------------------------------------------------- C2 + KATs

def test_c2_philox_full(shv, orc):
    w = W.C2
    f = Fam(shv, w.gen, w.seed, w.n_streams)
    got = f.gen_(w.n)
    same(got, f.ref(orc, w.n, offset=0))
    f.close()


def test_threefry_c2_shape_full_and_kats(shv, orc):
    """Threefry4x64-20 (NEXT-2): 2^16 counter-streams x 1024 u32 vs the oracle,
    and the Random123 KATs through the ABI (key = 4 words, ctr = (blk, g, 0, 0))."""
    f = Fam(shv, W.THREEFRY4X64_20, [12345, 6789, 42, 7], 1 << 16)
    ref = f.ref(orc, 1024, offset=0)
    same(f.gen_(1024), ref)
    f.close()
    rows = [ln.split() for ln in open(os.path.join(GOLD, "threefry4x64_kat.txt"))
            if ln.strip() and not ln.startswith("#")]
    for fam, *words in rows:
        v = [int(x, 16) for x in words]
        ctr, key, exp = v[0:4], v[4:8], v[8:12]
        if ctr[2] or ctr[3] or key[2] or key[3]:
            continue  # the ABI layout fixes ctr[2..3] = key[2..3] = 0
        seed = [key[0] & 0xFFFFFFFF, key[0] >> 32, key[1] & 0xFFFFFFFF, key[1] >> 32]
        h = shv.shv_streams_create_ex(W.THREEFRY4X64_20, seed, ctr[1], 1, 0, None, 0, -1, None)
        for _ in range(8):
            shv.shv_jump(h, shv.SHV_JUMP_DRAWS, ctr[0])
        out = torch.empty(8, dtype=torch.int32, device="cuda")
        shv.shv_generate_u32(h, out, 8, None)
        w = out.cpu().numpy().view(np.uint32).tolist()
        assert [w[2 * l] | (w[2 * l + 1] << 32) for l in range(4)] == exp, fam
        shv.shv_streams_destroy(h)


def test_philox_kats_through_abi(shv):
    rows = [ln.split() for ln in open(os.path.join(GOLD, "philox4x32_kat.txt"))
            if ln.strip() and not ln.startswith("#")]
    for fam, *words in rows:
        if fam != "philox4x32_10":
            continue
        v = [int(x, 16) for x in words]
        ctr, key, exp = v[0:4], v[4:6], v[6:10]
        g = ctr[2] | (ctr[3] << 32)
        blk = ctr[0] | (ctr[1] << 32)
        h = shv.shv_streams_create_ex(W.PHILOX4X32_10, key, g, 1, 0, None, 0, -1, None)
        for _ in range(4):  # offset 4*blk may exceed 2^64: jump in four parts
            shv.shv_jump(h, shv.SHV_JUMP_DRAWS, blk)
        out = torch.empty(4, dtype=torch.int32, device="cuda")
        shv.shv_generate_u32(h, out, 4, None)
        assert out.cpu().numpy().view(np.uint32).tolist() == exp, fam
        shv.shv_streams_destroy(h)


# ---------------------------------------------------------------- C3 (reduced, full compare)

@pytest.mark.parametrize("kind", ["u32", "f64", "f32"])
def test_c3_shape_reduced_full_compare(shv, orc, kind):
    f = Fam(shv, W.MRG32K3A, W.C3.seed, 1 << 12, W.SPACING_SUBSTREAM)
    ref = f.ref(orc, 4096, kind)
    same(f.gen_(4096, kind), ref)
    f.close()


# ---------------------------------------------------------------- edge cases

@pytest.mark.parametrize("gen,sp", [(W.MRG32K3A, 0), (W.MRG32K3A, 1), (W.PHILOX4X32_10, 0),
                                    (W.THREEFRY4X64_20, 0)])
@pytest.mark.parametrize("kind", ["u32", "f32", "f64"])
def test_ragged_offsets_and_replay(shv, orc, gen, sp, kind):
    """Rows that are not 32-byte multiples, offsets not multiples of 4 or 8,
    consecutive calls (offset advance), first_stream != 0, a single stream."""
    for ns, first in ((37, 5), (1, 0), (300, 1 << 40)):
        f = Fam(shv, gen, [12345] if gen == W.MRG32K3A else [12345, 777], ns, sp, first)
        for n in (1, 3, 8, 13, 64, 1000, 0, 7):
            before = f.offset
            got = f.gen_(n, kind)
            if n:
                same(got, f.ref(orc, n, kind, offset=before))
        f.close()


@pytest.mark.parametrize("kind", ["u32", "f32", "f64"])
def test_philox_keyed_mode(shv, orc, kind):
    """Parameterization (P L331-334): key = (first+i, tag), counter (blk, 0)."""
    for ns, first, n in ((300, 7, 1024), (33, (1 << 32) - 40, 13), (1, 0, 1000)):
        f = Fam(shv, W.PHILOX4X32_10, [0xABCD], ns, W.SPACING_KEYED, first)
        for pre in (0, 3):
            if pre:
                shv.shv_jump(f.h, shv.SHV_JUMP_DRAWS, pre)
                f.offset += pre
            before = f.offset
            same(f.gen_(n, kind), f.ref(orc, n, kind, offset=before))
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(ns, dtype=torch.int64, device="cuda")
        shv.shv_mc_pi_ex(f.h, 501, hits, cnt, None)
        torch.cuda.synchronize()
        tot, ref = orc.mc_count(W.PHILOX4X32_10, [0xABCD], ns, 501, first=first,
                                spacing=W.SPACING_KEYED, offset=f.offset)
        assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), ref) and int(hits.item()) == tot
        f.close()


@pytest.mark.parametrize("sp,seed", [(W.SPACING_STREAM, [12345, 9]), (W.SPACING_KEYED, [0xABCD])])
@pytest.mark.parametrize("kind,n", [("u32", 256), ("f32", 136), ("f64", 128), ("u32", 1024)])
def test_philox_short_rows_grouped_tasks(shv, orc, sp, seed, kind, n):
    """Many short rows (2^18 x <= 1 KB): the fast fill groups whole rows per
    warp task (PhiloxLaunch.rpt > 1); sampled rows and the jump-offset path."""
    ns = 1 << 18
    f = Fam(shv, W.PHILOX4X32_10, seed, ns, sp)
    rows = W.sample_streams(ns, 256, seed=11)
    try:
        for pre in (0, 4, 2):  # offset lane 0 (fast path), then lane 2 (generic path)
            if pre:
                shv.shv_jump(f.h, shv.SHV_JUMP_DRAWS, pre)
                f.offset += pre
            before = f.offset
            got = f.gen_(n, kind)
            same(got[rows], f.ref(orc, n, kind, offset=before, streams=rows))
    finally:
        f.close()


@pytest.mark.parametrize("gen,sp", [(W.MRG32K3A, 1), (W.PHILOX4X32_10, 0), (W.THREEFRY4X64_20, 0)])
def test_generate_twice_equals_generate_2n(shv, gen, sp):
    a = Fam(shv, gen, [99], 1000, sp)
    b = Fam(shv, gen, [99], 1000, sp)
    x1, x2 = a.gen_(512), a.gen_(512)
    y = b.gen_(1024)
    assert np.array_equal(np.concatenate([x1, x2], axis=1), y)
    # jump(k) then generate == generate and discard k
    c = Fam(shv, gen, [99], 1000, sp)
    shv.shv_jump(c.h, shv.SHV_JUMP_DRAWS, 300)
    assert np.array_equal(c.gen_(724), y[:, 300:])
    for f in (a, b, c):
        f.close()


def test_mrg_substream_and_stream_jumps(shv, orc):
    f = Fam(shv, W.MRG32K3A, [12345], 8, W.SPACING_SUBSTREAM)
    shv.shv_jump(f.h, shv.SHV_JUMP_SUBSTREAMS, 3)  # stream i -> substream i+3
    g = Fam(shv, W.MRG32K3A, [12345], 8, W.SPACING_SUBSTREAM, first=3)
    assert np.array_equal(f.gen_(64), g.gen_(64))
    shv.shv_jump(f.h, shv.SHV_JUMP_STREAMS, 1)
    pos = shv.shv_get_position(f.h)
    assert pos["offset"] == (1 << 127) + 3 * (1 << 76) + 64
    ref = orc.generate(W.MRG32K3A, [12345], 8, 16, spacing=1, offset=pos["offset"])
    same(f.gen_(16), ref)
    f.close()
    g.close()


def test_misaligned_output_and_errors(shv, orc):
    f = Fam(shv, W.PHILOX4X32_10, [5], 16)
    buf = torch.zeros(16 * 64 + 8, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(f.h, buf.data_ptr() + 4, 64, None)  # 4-byte aligned only
    torch.cuda.synchronize()
    got = buf.cpu().numpy().view(np.uint32)[1:1 + 16 * 64].reshape(16, 64)
    same(got, f.ref(orc, 64))
    f.offset += 64
    with pytest.raises(shv.ShvError) as ei:
        shv.shv_generate_u32(f.h, buf.data_ptr() + 2, 64, None)
    assert ei.value.status == shv.SHV_ERR_MISALIGNED
    with pytest.raises(shv.ShvError) as ei:
        shv.shv_generate_u32(f.h, 0, 64, None)
    assert ei.value.status == shv.SHV_ERR_INVALID_ARGUMENT
    shv.shv_generate_u32(f.h, 0, 0, None)  # n = 0: no-op
    assert shv.shv_get_position(f.h)["offset"] == 64
    hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(shv.ShvError) as ei:
        shv.shv_mc_pi(f.h, 0, hits, None)
    assert ei.value.status == shv.SHV_ERR_EMPTY_EXPERIMENT
    with pytest.raises(shv.ShvError) as ei:
        shv.shv_jump(f.h, shv.SHV_JUMP_SUBSTREAMS, 1)
    assert ei.value.status == shv.SHV_ERR_UNSUPPORTED
    f.close()
    with pytest.raises(shv.ShvError) as ei:
        f.close()
    assert ei.value.status == shv.SHV_ERR_LIFECYCLE


def test_short_form_create(shv, orc):
    h = shv.shv_streams_create(W.MRG32K3A, 12345, 4)
    out = torch.empty(4 * 1000, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, out, 1000, 0)
    torch.cuda.synchronize()
    same(out.cpu().numpy().view(np.uint32).reshape(4, 1000), orc.generate(W.MRG32K3A, [12345], 4, 1000))
    shv.shv_streams_destroy(h)


@pytest.mark.parametrize("gen,sp", [(W.MRG32K3A, 1), (W.PHILOX4X32_10, 0), (W.THREEFRY4X64_20, 0)])
def test_launch_config_invariance(shv, gen, sp):
    """R10: grid shape and segment length never change the values."""
    ref = None
    for bps, tpb, seg in ((0, 0, 0), (1, 32, 8), (3, 128, 64), (2, 256, 1024), (0, 64, 4096)):
        f = Fam(shv, gen, [31337], 777, sp)
        shv.shv_set_launch_config(f.h, bps, tpb, seg)
        x = np.concatenate([f.gen_(1000), f.gen_(24, "f64").view(np.uint32)], axis=1)
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(777, dtype=torch.int64, device="cuda")
        shv.shv_mc_pi_ex(f.h, 333, hits, cnt, None)
        torch.cuda.synchronize()
        res = (x, int(hits.item()), cnt.cpu().numpy())
        if ref is None:
            ref = res
        else:
            assert np.array_equal(res[0], ref[0]) and res[1] == ref[1]
            assert np.array_equal(res[2], ref[2])
        f.close()


def test_host_output_matches_device(shv, orc):
    # 40000 x 4000 u32 = 640 MB: three 256 MB staging slices, two in flight.
    for gen, sp, ns, n in ((W.MRG32K3A, 1, 40000, 4000), (W.PHILOX4X32_10, 0, 3000, 2000)):
        a = Fam(shv, gen, [4242], ns, sp)
        b = Fam(shv, gen, [4242], ns, sp)
        host = torch.empty(ns * n, dtype=torch.int32, pin_memory=True)
        shv.shv_generate_u32_host(a.h, host, n, None)
        torch.cuda.synchronize()
        dev = b.gen_(n)
        assert np.array_equal(host.numpy().view(np.uint32).reshape(ns, n), dev)
        assert shv.shv_get_position(a.h)["offset"] == n
        a.close()
        b.close()


# ---------------------------------------------------------------- Monte Carlo

@pytest.mark.parametrize("gen,sp", [(W.MRG32K3A, 1), (W.PHILOX4X32_10, 0), (W.THREEFRY4X64_20, 0)])
def test_mc_counts_small_full(shv, orc, gen, sp):
    f = Fam(shv, gen, [12345], 300, sp, first=17)
    for samples, pre in ((1000, 0), (777, 1), (5, 3), (4096, 2)):
        if pre:
            shv.shv_jump(f.h, shv.SHV_JUMP_DRAWS, pre)
            f.offset += pre
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(300, dtype=torch.int64, device="cuda")
        shv.shv_mc_pi_ex(f.h, samples, hits, cnt, None)
        torch.cuda.synchronize()
        tot, ref = orc.mc_count(gen, [12345], 300, samples, first=17, spacing=sp, offset=f.offset)
        f.offset += 2 * samples
        assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), ref)
        assert int(hits.item()) == tot
    f.close()


# Seeds whose first step hits the edges of the FP64 floor reductions
# (tests/test_fp64_step_bounds.py): component 1 at residue 0 with p < 0 (the
# step carries r = m1) together with component 2 at residue 0 (a tie, z = m1);
# both components at residue m - 1; SURVEY App. A.1's tie state.
EDGE_SEEDS = [
    [4294809486, 2474611487, 12345, 0, 1, 0],
    [4294967086, 3588371285, 7, 0, 5, 4239484263],
    [0, 1, 0, 0, 0, 1226359468],
]


@pytest.mark.parametrize("seed", EDGE_SEEDS)
def test_mrg_fp64_step_edge_states(shv, orc, seed):
    for n, kind in ((64, "u32"), (37, "u32"), (64, "f32"), (32, "f64")):
        f = Fam(shv, W.MRG32K3A, seed, 3, 0)
        got = f.gen_(n, kind)
        same(got, f.ref(orc, n, kind, offset=0))
        f.close()
    z0 = orc.generate(W.MRG32K3A, seed, 1, 1)[0, 0]
    assert seed != EDGE_SEEDS[0] or z0 == M1  # the tie
    f = Fam(shv, W.MRG32K3A, seed, 3, 0)
    hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
    shv.shv_mc_pi_ex(f.h, 100, hits, cnt, None)
    torch.cuda.synchronize()
    tot, ref = orc.mc_count(W.MRG32K3A, seed, 3, 100)
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), ref) and int(hits.item()) == tot
    f.close()


# ---------------------------------------------------------------- full BASELINE sizes

def _golden_full():
    p = os.path.join(GOLD, "oracle_full.json")
    if not os.path.exists(p):
        pytest.skip("tests/golden/oracle_full.json not generated")
    return json.load(open(p))


def _checksums_gpu(t_u32: torch.Tensor, n: int, t_f64=None):
    """Test-side reductions of a GPU output (the same aggregates make_golden.py
    computes with the oracle): sum, weighted XOR over J = i*n + j, ties."""
    v = t_u32.view(-1)
    N = v.numel()
    sum_z, wx, ties, sum_f = 0, 0, 0, 0
    CH = 1 << 27
    for s in range(0, N, CH):
        x = v[s:s + CH].to(torch.int64) & 0xFFFFFFFF
        J = torch.arange(s, s + x.numel(), device=x.device, dtype=torch.int64)
        sum_z += int(x.sum().item()) & ((1 << 64) - 1)
        ties += int((x == M1).sum().item())
        p = x * (2 * J + 1)  # wraps mod 2^64 in two's complement
        while p.numel() > 1:
            if p.numel() & 1:
                p = torch.cat([p, torch.zeros(1, dtype=p.dtype, device=p.device)])
            p = torch.bitwise_xor(p[0::2], p[1::2])
        wx ^= int(p.item()) & ((1 << 64) - 1)
        if t_f64 is not None:
            sum_f += int(t_f64.view(-1)[s:s + CH].view(torch.int64).sum().item())
        del x, J, p
    return sum_z % (1 << 64), "%016x" % wx, ties, "%016x" % (sum_f % (1 << 64))


def test_c2_checksums(shv):
    g = _golden_full()
    if "C2_u32" not in g:
        pytest.skip("C2 checksums not generated")
    w = W.C2
    f = Fam(shv, w.gen, w.seed, w.n_streams)
    out = torch.empty(w.n_streams * w.n, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(f.h, out, w.n, None)
    sz, wx, _, _ = _checksums_gpu(out, w.n)
    assert (sz, wx) == (g["C2_u32"]["sum_z"], g["C2_u32"]["wxor"])
    f.close()


def test_c3_full_size_sampled_and_checksums(shv, orc):
    """2^20 substreams x 4096 (u32 and f64): sampled rows vs oracle, plus
    whole-output checksums vs tests/golden/oracle_full.json."""
    w = W.C3
    streams = W.sample_streams(w.n_streams, 512)
    a = Fam(shv, w.gen, w.seed, w.n_streams, w.spacing)
    out = torch.empty(w.n_streams * w.n, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(a.h, out, w.n, None)
    torch.cuda.synchronize()
    idx = torch.tensor(streams, device="cuda")
    rows = out.view(w.n_streams, w.n)[idx].cpu().numpy().view(np.uint32)
    same(rows, orc.generate(w.gen, list(w.seed), 0, w.n, spacing=w.spacing, streams=streams))
    b = Fam(shv, w.gen, w.seed, w.n_streams, w.spacing)
    out64 = torch.empty(w.n_streams * w.n, dtype=torch.float64, device="cuda")
    shv.shv_generate_f64(b.h, out64, w.n, None)
    torch.cuda.synchronize()
    rows64 = out64.view(w.n_streams, w.n)[idx].cpu().numpy()
    same(rows64, orc.generate(w.gen, list(w.seed), 0, w.n, spacing=w.spacing, streams=streams,
                              kind=2))
    g = _golden_full().get("C3")
    if g:
        sz, wx, ties, sf = _checksums_gpu(out, w.n, out64)
        assert (sz, wx, ties, sf) == (g["sum_z"], g["wxor"], g["ties"], g["sum_f64_bits"])
    a.close()
    b.close()


@pytest.mark.parametrize("w", [W.C4_MRG, W.C4_PHILOX], ids=["mrg", "philox"])
def test_c4_mc_pi_full_size(shv, orc, w):
    """2^38 samples over 2^20 streams: sampled per-stream counts vs oracle,
    total vs oracle total (golden), pi within the 4-sigma binomial bound."""
    f = Fam(shv, w.gen, w.seed, w.n_streams, w.spacing)
    hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(w.n_streams, dtype=torch.int64, device="cuda")
    shv.shv_mc_pi_ex(f.h, w.n, hits, cnt, None)
    torch.cuda.synchronize()
    total = int(hits.item())
    counts = cnt.cpu().numpy().astype(np.uint64)
    assert int(counts.sum()) == total
    streams = W.sample_streams(w.n_streams, 1024)  # >= 1024 sampled streams
    _, ref = orc.mc_count(w.gen, list(w.seed), 0, w.n, spacing=w.spacing, streams=streams)
    assert np.array_equal(counts[streams], ref)
    N = w.n_streams * w.n
    p = 221069946527026 / 2 ** 48
    assert abs(4 * total / N - math.pi) <= 4 * 4 * math.sqrt(p * (1 - p) / N)
    key = "C4_mrg_total" if w.gen == W.MRG32K3A else "C4_philox_total"
    g = _golden_full()
    if key in g:
        assert total == g[key]
    f.close()


@pytest.mark.parametrize("w", [W.C5_MRG, W.C5_PHILOX], ids=["mrg", "philox"])
def test_c5_rank_slices_match(shv, orc, w):
    """Weak-scaling shards (rank r fills streams [r*2^20, (r+1)*2^20)): sampled
    rows of rank 3 of 8 at full size vs the oracle, in bench.py's launch
    configuration."""
    ws = W.rank_slice(w, 3, 8, weak=True)
    f = Fam(shv, ws.gen, ws.seed, ws.n_streams, ws.spacing, ws.first)
    out = torch.empty(ws.n_streams * ws.n, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(f.h, out, ws.n, None)
    torch.cuda.synchronize()
    streams = W.sample_streams(ws.n_streams, 256)
    rows = out.view(ws.n_streams, ws.n)[torch.tensor(streams, device="cuda")].cpu().numpy()
    same(rows.view(np.uint32), orc.generate(ws.gen, list(ws.seed), 0, ws.n, first=ws.first,
                                            spacing=ws.spacing, streams=streams))
    f.close()


def test_concurrent_handles_from_threads(shv, orc):
    """The registry is mutex-protected (include/shv.h): host threads creating,
    filling (each on its own CUDA stream) and destroying handles concurrently
    get exactly their own streams' values."""
    import threading
    results, errors = {}, []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                gen = (W.MRG32K3A, W.PHILOX4X32_10, W.THREEFRY4X64_20)[k % 3]
                st = torch.empty(6 * 64, dtype=torch.int32, device="cuda") if gen == W.MRG32K3A else None
                for rep in range(5):
                    h = shv.shv_streams_create_ex(gen, [1000 + k], 64 * k, 64, 0, st, 0, -1, s)
                    out = torch.empty(64 * 96, dtype=torch.int32, device="cuda")
                    shv.shv_generate_u32(h, out, 96, s)
                    s.synchronize()
                    shv.shv_streams_destroy(h)
                results[k] = (gen, out.cpu().numpy().view(np.uint32).reshape(64, 96))
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(9)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k, (gen, got) in results.items():
        same(got, orc.generate(gen, [1000 + k], 64, 96, first=64 * k))


# --------------------------------------------------------------------------- index-space extremes
# The last streams of each family at offsets just below each generator's
# exhaustion point: every 64/128-bit carry in the kernels' counter and
# position arithmetic (P L264-268; R4, R6, R13, R16) against the oracle.
# Offsets are reached with shv_jump: (kind, count) pairs.

U64 = (1 << 64) - 1


@pytest.mark.parametrize("gen,seed,spacing,first,ns,jumps,m", [
    (W.MRG32K3A, [12345], W.SPACING_STREAM, (1 << 64) - 3, 3, [(1, (1 << 51) - 1), (0, U64 - 4)], 200),
    (W.MRG32K3A, [7, 8, 9, 10, 11, 12], W.SPACING_SUBSTREAM, (1 << 51) - 4, 4, [(2, 1), (1, 5), (0, U64)], 160),
    (W.PHILOX4X32_10, [0xFFFFFFFF, 0xFFFFFFFF], W.SPACING_STREAM, (1 << 64) - 5, 5,
     [(0, U64)] * 3 + [(0, U64 - 400)], 200),
    (W.PHILOX4X32_10, [99], W.SPACING_KEYED, (1 << 32) - 3, 3, [(0, U64)] * 3 + [(0, U64 - 197)], 96),
    (W.THREEFRY4X64_20, [1, 2, 3, 4], W.SPACING_STREAM, (1 << 64) - 2, 2, [(0, U64)] * 7 + [(0, U64 - 293)], 128),
])
def test_index_space_extremes(shv, orc, gen, seed, spacing, first, ns, jumps, m):
    st = torch.empty(6 * ns, dtype=torch.int32, device="cuda") if gen == W.MRG32K3A else None
    h = shv.shv_streams_create_ex(gen, seed, first, ns, spacing, st, 0, torch.cuda.current_device(), None)
    for kind, count in jumps:
        shv.shv_jump(h, kind, count)
    for kind, dt, ndt in ((0, torch.int32, np.uint32), (2, torch.float64, np.float64)):
        mm = m // 2 if (kind == 2 and gen != W.MRG32K3A) else m
        out = torch.empty(ns * mm, dtype=dt, device="cuda")
        pos = shv.shv_get_position(h)["offset"]
        getattr(shv, "shv_generate_" + ("u32" if kind == 0 else "f64"))(h, out, mm, None)
        torch.cuda.synchronize()
        want = orc.generate(gen, seed, ns, mm, first=first, spacing=spacing, offset=pos, kind=kind)
        got = out.cpu().numpy().view(ndt).reshape(ns, mm)
        assert np.array_equal(got.view(np.uint8), np.ascontiguousarray(want).view(np.uint8)), (gen, kind)
    if gen != W.MRG32K3A:  # the counter-based streams are now (nearly) exhausted
        out = torch.empty(ns * 64, dtype=torch.int32, device="cuda")
        with pytest.raises(shv.ShvError) as e:
            shv.shv_generate_u32(h, out, 64, None)
        assert e.value.status == shv.SHV_ERR_INVALID_ARGUMENT
    shv.shv_streams_destroy(h)


def _full_compare(shv, orc, w, kind):
    """Every value of a BASELINE full-size workload against the oracle, in
    2^16-stream chunks (device -> host copy per chunk; the oracle on all host
    cores)."""
    fam = Fam(shv, w.gen, w.seed, w.n_streams, w.spacing, w.first)
    dt, ndt = (torch.int32, np.uint32) if kind == 0 else (torch.float64, np.float64)
    out = torch.empty(w.n_streams * w.n, dtype=dt, device="cuda")
    (shv.shv_generate_u32 if kind == 0 else shv.shv_generate_f64)(fam.h, out, w.n, None)
    torch.cuda.synchronize()
    rows = out.view(w.n_streams, w.n)
    step = 1 << 16
    for s0 in range(0, w.n_streams, step):
        got = rows[s0:s0 + step].cpu().numpy().view(ndt)
        want = orc.generate(w.gen, list(w.seed), step, w.n, first=w.first + s0, spacing=w.spacing, kind=kind)
        assert np.array_equal(got.view(np.uint8), np.ascontiguousarray(want).view(np.uint8)), (w.name, kind, s0)
    fam.close()
    del out


@pytest.mark.parametrize("w,kind", [(W.C3, 0), (W.C3, 2), (W.C5_PHILOX, 0)], ids=["c3-u32", "c3-f64", "c5-philox-u32"])
def test_full_size_every_value(shv, orc, w, kind):
    """C3 (2^20 MRG32k3a substreams x 4096, u32 and f64) and the C5 Philox
    rank-0 slice (2^20 counter-streams x 4096): all 2^32 values of each,
    element by element, in the launch configuration bench.py times."""
    _full_compare(shv, orc, w, kind)
