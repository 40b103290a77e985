"""GPU parity for the disjointness audit (SPEC verify_disjoint, S L407-415,
L425-426): shv_verify_disjoint (kernels_audit.cu, hash
table in HBM) against oracle.verify_disjoint (a plain dict of windows). The
report is integer work, compared field by field, bit-exact.
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


def audit(shv, rows_dev, n_pe, horizon, ws_bytes=None):
    need = shv.shv_verify_disjoint_workspace_bytes(n_pe, horizon)
    ws_bytes = need if ws_bytes is None else ws_bytes
    ws = torch.empty(max(ws_bytes, 8) // 8, dtype=torch.int64, device="cuda")
    rep = torch.zeros(7, dtype=torch.int64, device="cuda")
    shv.shv_verify_disjoint(rows_dev, n_pe, horizon, ws, ws_bytes, rep)
    torch.cuda.synchronize()
    v = [int(x) & ((1 << 64) - 1) for x in rep.cpu().tolist()]
    return dict(zip(shv.DISJOINT_REPORT_FIELDS, v))


def expect(orc_report):
    none = (1 << 64) - 1
    r = {"disjoint": int(orc_report["disjoint"]), "windows": orc_report["windows"],
         "colliding": orc_report["colliding"]}
    for k in ("pe_a", "pos_a", "pe_b", "pos_b"):
        r[k] = orc_report.get(k, none)
    return r


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def gen_rows(shv, gen, seed, n, m, first=0, spacing=W.SPACING_STREAM, jump=0):
    h = shv.shv_streams_create_ex(gen, seed, first, n, spacing, None, 0, torch.cuda.current_device(), None)
    if jump:
        shv.shv_jump(h, shv.SHV_JUMP_DRAWS, jump)
    out = torch.empty(n * m, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, out, m, None)
    torch.cuda.synchronize()
    shv.shv_streams_destroy(h)
    return out


@pytest.mark.parametrize("alphabet", [2, 3, 7, 1 << 32])
def test_random_rows_match_oracle(shv, orc, alphabet):
    """Small alphabets: many equal windows within and across PEs, ties, repeats."""
    rng = np.random.default_rng(alphabet)
    for trial in range(12):
        n_pe = int(rng.integers(1, 9))
        horizon = int(rng.integers(1, 300))
        rows = rng.integers(0, alphabet, size=(n_pe, horizon), dtype=np.uint64).astype(np.uint32)
        got = audit(shv, to_dev(rows), n_pe, horizon)
        assert got == expect(orc.verify_disjoint(list(rows))), (alphabet, trial, n_pe, horizon)


def test_degenerate_shapes(shv, orc):
    # no windows (horizon < 4, or no PEs): disjoint, NULL rows allowed
    for n_pe, horizon in ((0, 100), (5, 0), (5, 3)):
        rep = torch.zeros(7, dtype=torch.int64, device="cuda")
        shv.shv_verify_disjoint(None, n_pe, horizon, None, 0, rep)
        torch.cuda.synchronize()
        r = dict(zip(shv.DISJOINT_REPORT_FIELDS, [int(x) & ((1 << 64) - 1) for x in rep.cpu().tolist()]))
        assert r["disjoint"] == 1 and r["windows"] == 0 and r["colliding"] == 0
        assert r["pe_a"] == (1 << 64) - 1
    # one PE: repeats inside a row are not collisions
    rows = np.zeros((1, 50), dtype=np.uint32)
    assert audit(shv, to_dev(rows), 1, 50) == expect(orc.verify_disjoint(list(rows)))
    # every PE identical and constant: one value, maximal contention on one slot
    rows = np.zeros((64, 1000), dtype=np.uint32)
    got = audit(shv, to_dev(rows), 64, 1000)
    assert got == {"disjoint": 0, "windows": 64 * 997, "colliding": 1,
                   "pe_a": 0, "pos_a": 0, "pe_b": 1, "pos_b": 0}


def test_workspace_size_does_not_change_the_report(shv, orc):
    rng = np.random.default_rng(11)
    rows = rng.integers(0, 3, size=(6, 200)).astype(np.uint32)
    want = expect(orc.verify_disjoint(list(rows)))
    d = to_dev(rows)
    need = shv.shv_verify_disjoint_workspace_bytes(6, 200)
    for extra in (0, 8, 4096, 1 << 20):
        assert audit(shv, d, 6, 200, ws_bytes=need + extra) == want, extra


def test_many_buckets_match_oracle(shv, orc):
    """> 2^16 windows: the radix partition uses several buckets (2^17 windows -> 2
    buckets, 2^19 -> 8); small alphabet so collisions land in many buckets."""
    rng = np.random.default_rng(3)
    for n_pe, horizon, alphabet in ((256, 515, 2), (64, 8195, 5), (8, 65539, 1 << 32)):
        rows = rng.integers(0, alphabet, size=(n_pe, horizon), dtype=np.uint64).astype(np.uint32)
        if alphabet == 1 << 32:  # plant overlaps between rows 6 -> 2 and 7 -> 5
            rows[2, 1000:1010] = rows[6, 50000:50010]
            rows[5, 7:9000] = rows[7, 100:9093]
        got = audit(shv, to_dev(rows), n_pe, horizon)
        assert got == expect(orc.verify_disjoint(list(rows))), (n_pe, horizon, alphabet)


def test_errors(shv):
    d = to_dev(np.zeros((2, 10), dtype=np.uint32))
    rep = torch.zeros(7, dtype=torch.int64, device="cuda")
    need = shv.shv_verify_disjoint_workspace_bytes(2, 10)
    # 14 windows, one bucket: 6 scratch + 5 per-bucket + 6 per-window u64 words
    assert need == 8 * (6 + 5 + 6 * 14)
    ws = torch.empty(need // 8 + 8, dtype=torch.int64, device="cuda")
    with pytest.raises(shv.ShvError) as e:  # one word short
        shv.shv_verify_disjoint(d, 2, 10, ws, need - 8, rep)
    assert e.value.status == shv.SHV_ERR_INVALID_ARGUMENT
    with pytest.raises(shv.ShvError) as e:
        shv.shv_verify_disjoint(d, 2, 10, ws.data_ptr() + 4, need, rep)
    assert e.value.status == shv.SHV_ERR_MISALIGNED
    with pytest.raises(shv.ShvError) as e:
        shv.shv_verify_disjoint(d, 2, 10, ws, need, rep.data_ptr() + 4)
    assert e.value.status == shv.SHV_ERR_MISALIGNED
    with pytest.raises(shv.ShvError) as e:
        shv.shv_verify_disjoint(d, 1 << 20, 1 << 20, ws, need, rep)
    assert e.value.status == shv.SHV_ERR_INVALID_ARGUMENT
    with pytest.raises(shv.ShvError) as e:
        shv.shv_verify_disjoint(None, 2, 10, ws, need, rep)
    assert e.value.status == shv.SHV_ERR_INVALID_ARGUMENT
    assert shv.shv_verify_disjoint_workspace_bytes(1 << 20, 1 << 21) == 0
    assert shv.shv_verify_disjoint_workspace_bytes(5, 3) == 0  # no windows, no workspace


def test_spec_examples_on_generated_rows(shv, orc):
    # S L412: MRG32k3a Sequence Splitting, 8 PEs, horizon 10^5 -> disjoint
    rows = gen_rows(shv, W.MRG32K3A, [12345], 8, 100000)
    got = audit(shv, rows, 8, 100000)
    assert got["disjoint"] == 1 and got["windows"] == 8 * 99997 and got["colliding"] == 0
    # S L414: a deliberately overlapping plan -> collision at position 0
    a = gen_rows(shv, W.PHILOX4X32_10, [7], 4, 200)
    b = gen_rows(shv, W.PHILOX4X32_10, [7], 4, 200, first=2)
    both = torch.cat([a, b])
    want = expect(orc.verify_disjoint(list(orc.generate(W.PHILOX4X32_10, [7], 4, 200))
                                      + list(orc.generate(W.PHILOX4X32_10, [7], 4, 200, first=2))))
    got = audit(shv, both, 8, 200)
    assert got == want and (got["pe_a"], got["pos_a"], got["pe_b"], got["pos_b"]) == (2, 0, 4, 0)
    # shifted overlap: stream 1 jumped by 17 draws sits inside stream 1's row
    c = gen_rows(shv, W.MRG32K3A, [12345], 4, 300)
    d = gen_rows(shv, W.MRG32K3A, [12345], 1, 300, first=1, jump=17)
    got = audit(shv, torch.cat([c, d]), 5, 300)
    assert (got["disjoint"], got["pe_a"], got["pos_a"], got["pe_b"], got["pos_b"]) == (0, 1, 17, 4, 0)
    assert got["colliding"] == 300 - 17 - 3
    # S L415: LeapFrog{2}, horizon 10^4 -> disjoint
    h = shv.shv_streams_create_leapfrog(W.MRG32K3A, [12345], 2, 0, 2, None, 0, torch.cuda.current_device(), None)
    out = torch.empty(2 * 10000, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, out, 10000, None)
    shv.shv_streams_destroy(h)
    assert audit(shv, out, 2, 10000)["disjoint"] == 1


def test_c3_prefix_disjoint_and_planted_collision(shv):
    """BASELINE C3 layout (MRG32k3a substreams of seed 12345) at 2^18 x 4096:
    ~1.07e9 windows, disjoint by construction (distinct jump exponents, S L179);
    then one planted 4-word copy is found exactly, wherever it is."""
    n, m = 1 << 18, 4096
    rows = gen_rows(shv, W.MRG32K3A, [12345], n, m, spacing=W.SPACING_SUBSTREAM)
    got = audit(shv, rows, n, m)
    assert got["disjoint"] == 1 and got["windows"] == n * (m - 3) and got["colliding"] == 0
    r2 = rows.view(n, m)
    r2[200000, 3000:3004] = r2[1000, 77:81]
    got = audit(shv, rows, n, m)
    assert (got["disjoint"], got["colliding"], got["pe_a"], got["pos_a"], got["pe_b"], got["pos_b"]) == \
        (0, 1, 1000, 77, 200000, 3000)
    del rows
    torch.cuda.empty_cache()
