"""GPU parity of the MRG32k3a row-tile fill (mrg_fill_rows_kernel).

The row-tile path covers the C3/C5 shapes at the default launch configuration
(tests/test_gpu_parity.py compares those). Here small shapes are forced onto it
by shrinking the resident grid (1 block of 32 threads per SM: the path is taken
when there are at least 2 tiles of 32 segments per resident warp), and every
value is compared with the oracle: segment lengths S = 128, 96, 160; rows of
fewer than 32 segments (tiles spanning several rows), of exactly 32, and of more
than 32 (nseg 33 / 80: the per-tile (A^(32 S))^(j / 32) jumps; nseg a multiple of
32: run mode, where a warp carries its lanes from tile to tile by A^(31 S), with a
ragged last run at 86 tiles per row); a ragged last tile; non-zero offsets;
STREAM and SUBSTREAM spacing with first > 0; u32, f32 and f64 (f64 segments hold half the values:
the same 512-B segments). A CUDA profiler trace
checks that the row-tile kernel is the one that ran.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def shv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1412_8266_b200 as shv
    return shv


@pytest.fixture(scope="module")
def orc():
    import oracle
    return oracle


def kernels_of(fn):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        fn()
        torch.cuda.synchronize()
    return [e.name for e in p.events() if e.device_type.name == "CUDA"]


CASES = [
    # (n_streams, n, spacing, first, pre_offset); S = mrg_rows_seg_len(n): 128, 96, 160, ... (first divisor)
    (600, 4096, W.SPACING_SUBSTREAM, 0, 0),        # S 128, nseg 32: a tile = one row (the C5 layout)
    (600, 2048, W.SPACING_STREAM, 0, 3),           # S 128, nseg 16: a tile = two rows
    (601, 4096, W.SPACING_SUBSTREAM, 7, 1000),     # ragged last tile, offset 1000, first 7
    (300, 8192, W.SPACING_STREAM, 3, 17),          # S 128, nseg 64: run mode, 2 tiles per row
    (240, 256 * 40, W.SPACING_STREAM, 2, 9),       # S 128, nseg 80: segments j >= 32 by per-tile per-bit jumps
    (300, 128 * 33, W.SPACING_SUBSTREAM, 1, 4),    # S 128, nseg 33
    (70, 256 * 160, W.SPACING_SUBSTREAM, 0, 5),    # S 128, nseg 320: run mode, 10 tiles per row
    (3201, 384, W.SPACING_SUBSTREAM, 11, 0),       # S 128, nseg 3: tiles span rows, ragged
    (2000, 480, W.SPACING_STREAM, 0, 33),          # S 96
    (1400, 1120, W.SPACING_SUBSTREAM, 0, 0),       # S 160
    (64, 8192 * 43, W.SPACING_SUBSTREAM, 5, 77),   # S 128, run mode: 86 tiles per row, runs of 9 (last 5)
]


@pytest.mark.parametrize("ns,n,spacing,first,pre", CASES)
@pytest.mark.parametrize("kind", ["u32", "f32", "f64"])
def test_rows_fill_matches_oracle(shv, orc, ns, n, spacing, first, pre, kind):
    st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
    h = shv.shv_streams_create_ex(W.MRG32K3A, [12345, 777, 31337, 4242, 99, 5], first, ns, spacing, st, 0,
                                  torch.cuda.current_device(), None)
    try:
        shv.shv_set_launch_config(h, 1, 32, 0)
        if pre:
            shv.shv_jump(h, 0, pre, None)
        tdt = {"u32": torch.int32, "f32": torch.float32, "f64": torch.float64}[kind]
        okind = {"u32": 0, "f32": 1, "f64": 2}[kind]
        vdt = np.uint64 if kind == "f64" else np.uint32
        out = torch.empty(ns * n, dtype=tdt, device="cuda")
        names = kernels_of(lambda: getattr(shv, "shv_generate_" + kind)(h, out, n, None))
        assert any("mrg_fill_rows_kernel" in k for k in names), names
        got = out.cpu().numpy().view(vdt).reshape(ns, n)
        ref = orc.generate(W.MRG32K3A, [12345, 777, 31337, 4242, 99, 5], ns, n, first=first, spacing=spacing,
                           offset=pre, kind=okind)
        ref = np.ascontiguousarray(ref).view(vdt).reshape(ns, n)
        bad = np.nonzero(got != ref)
        assert len(bad[0]) == 0, f"{len(bad[0])} mismatches, first at {[x[:5] for x in bad]}"
        # the handle advanced by n: a second call continues the streams
        out2 = torch.empty(ns * 256, dtype=tdt, device="cuda")
        getattr(shv, "shv_generate_" + kind)(h, out2, 256, None)
        ref2 = orc.generate(W.MRG32K3A, [12345, 777, 31337, 4242, 99, 5], ns, 256, first=first, spacing=spacing,
                            offset=pre + n, kind=okind)
        assert np.array_equal(out2.cpu().numpy().view(vdt).reshape(ns, 256),
                              np.ascontiguousarray(ref2).view(vdt).reshape(ns, 256))
    finally:
        shv.shv_streams_destroy(h)


def test_rows_path_not_taken_for_few_tiles(shv):
    """At the default launch configuration a small shape keeps the stream-per-lane TMA path."""
    ns, n = 64, 4096
    st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
    h = shv.shv_streams_create_ex(W.MRG32K3A, [12345], 0, ns, W.SPACING_SUBSTREAM, st, 0,
                                  torch.cuda.current_device(), None)
    try:
        out = torch.empty(ns * n, dtype=torch.int32, device="cuda")
        names = kernels_of(lambda: shv.shv_generate_u32(h, out, n, None))
        assert not any("mrg_fill_rows_kernel" in k for k in names), names
        assert any("mrg_fill_tma_kernel" in k for k in names), names
    finally:
        shv.shv_streams_destroy(h)


def test_rows_fill_component1_edge_state(shv, orc):
    """MrgMF's component-1 edge: a negative product sum that is an exact multiple
    of m1 floors to k - 1 and leaves the residue m1 (= 0) as the next state word. The seed puts
    it on the first step of stream 0 (x1 = 1, x0 = a12 / a13n mod m1, so a12 x1 - a13n x0 = k m1 < 0);
    every value of the row-tile fill, and the fused MC totals, must equal the oracle's."""
    M1, A12, A13N = 4294967087, 1403580, 810728
    x0 = A12 * pow(A13N, -1, M1) % M1
    assert (A12 * 1 - A13N * x0) % M1 == 0 and A12 - A13N * x0 < 0
    seed = [x0, 1, 12345, 777, 31337, 4242]
    ns, n = 600, 4096
    st = torch.empty(6 * ns, dtype=torch.int32, device="cuda")
    h = shv.shv_streams_create_ex(W.MRG32K3A, seed, 0, ns, W.SPACING_SUBSTREAM, st, 0, torch.cuda.current_device(), None)
    try:
        shv.shv_set_launch_config(h, 1, 32, 0)
        out = torch.empty(ns * n, dtype=torch.int32, device="cuda")
        names = kernels_of(lambda: shv.shv_generate_u32(h, out, n, None))
        assert any("mrg_fill_rows_kernel" in k for k in names), names
        ref = orc.generate(W.MRG32K3A, seed, ns, n, first=0, spacing=W.SPACING_SUBSTREAM, offset=0, kind=0)
        got = out.cpu().numpy().view(np.uint32).reshape(ns, n)
        assert np.array_equal(got, np.ascontiguousarray(ref).view(np.uint32).reshape(ns, n))
    finally:
        shv.shv_streams_destroy(h)
    h = shv.shv_streams_create_ex(W.MRG32K3A, seed, 0, ns, W.SPACING_SUBSTREAM, st, 0, torch.cuda.current_device(), None)
    try:
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(ns, dtype=torch.int64, device="cuda")
        shv.shv_mc_pi_ex(h, n, hits, cnt, None)
        torch.cuda.synchronize()
        tot, cref = orc.mc_count(W.MRG32K3A, seed, ns, n, spacing=W.SPACING_SUBSTREAM)
        assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), cref) and int(hits.item()) == tot
    finally:
        shv.shv_streams_destroy(h)
