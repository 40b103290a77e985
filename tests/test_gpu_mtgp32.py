"""GPU parity for MTGP32-11213 handles (NEXT-4c; [Saito.Matsumoto2012] via
P L74-76 [§2.2], L133-136 [§2.3]; R18): the block-cooperative sm_100a kernel
(kernels_mtgp32.cu) against the oracle's sequential recursion
(oracle/shv_oracle.c orc_mtgp32_*), bit-exact for every kind, across calls,
jumps, stream subsets, host output and the fused Monte Carlo count.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

DT = {"u32": (torch.int32, np.uint32, 0), "f32": (torch.float32, np.float32, 1),
      "f64": (torch.float64, np.float64, 2)}


@pytest.fixture(scope="module")
def shv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1412_8266_b200 as shv
    return shv


@pytest.fixture(scope="module")
def params():
    return W.mtgp32_params()


class Mt:
    def __init__(self, shv, params, seed, first, n):
        self.shv, self.params, self.seed, self.first, self.n = shv, params, seed, first, n
        self.h = shv.shv_streams_create_mtgp32(params, seed, first, n, None, 0, torch.cuda.current_device(), None)
        self.offset = 0

    def gen(self, m, kind="u32", host=False):
        tdt, ndt, _ = DT[kind]
        if host:
            out = torch.empty(self.n * m, dtype=tdt, pin_memory=True)
            self.shv.shv_generate_u32_host(self.h, out, m, None)
        else:
            out = torch.empty(self.n * m, dtype=tdt, device="cuda")
            getattr(self.shv, "shv_generate_" + kind)(self.h, out, m, None)
        torch.cuda.synchronize()
        self.offset += m * (2 if kind == "f64" else 1)
        return out.cpu().numpy().view(ndt).reshape(self.n, m)

    def ref(self, orc, m, kind="u32", streams=None, offset=None):
        return orc.generate(W.MTGP32, W.mtgp32_seed_words(self.seed, self.params), self.n, m, first=self.first,
                            offset=self.offset if offset is None else offset, kind=DT[kind][2], streams=streams)

    def close(self):
        self.shv.shv_streams_destroy(self.h)


def test_all_200_streams_u32(shv, orc, params):
    mt = Mt(shv, params, 12345, 0, 200)
    want = mt.ref(orc, 5000)
    got = mt.gen(5000)
    assert (got == want).all()
    mt.close()


@pytest.mark.parametrize("kind", ["u32", "f32", "f64"])
def test_kinds_and_call_sequences(shv, orc, params, kind):
    """Ragged lengths (partial rounds, n below one round, n = 1), successive
    calls continuing each other, every kind."""
    mt = Mt(shv, params, 7, 13, 40)
    for m in (1, 255, 256, 257, 1000, 3, 4099):
        want = mt.ref(orc, m, kind)
        got = mt.gen(m, kind)
        assert (got == want).all() if kind == "u32" else np.array_equal(got, want), (kind, m)
    mt.close()


def test_jump_and_offsets(shv, orc, params):
    mt = Mt(shv, params, (1 << 40) + 3, 100, 64)
    mt.gen(77)
    shv.shv_jump(mt.h, shv.SHV_JUMP_DRAWS, 5001)
    mt.offset += 5001
    torch.cuda.synchronize()
    want = mt.ref(orc, 2048)
    assert (mt.gen(2048) == want).all()
    assert shv.shv_get_position(mt.h)["offset"] == 77 + 5001 + 2048
    with pytest.raises(shv.ShvError) as e:
        shv.shv_jump(mt.h, shv.SHV_JUMP_SUBSTREAMS, 1)
    assert e.value.status == shv.SHV_ERR_UNSUPPORTED
    mt.close()


def test_more_states_than_resident_ctas(shv, orc, params):
    """2000 states (parameter records repeated: test-only, not independent
    streams) > 148 x 8 resident CTAs: CTAs loop over states."""
    P = [params[g % 200] for g in range(2000)]
    mt = Mt(shv, P, 99, 0, 2000)
    idx = W.sample_streams(2000, 64)
    want = mt.ref(orc, 600, streams=idx)
    got = mt.gen(600)
    assert (got[idx] == want).all()
    mt.close()


def test_host_output(shv, orc, params):
    mt = Mt(shv, params, 5, 0, 200)
    want = mt.ref(orc, 3000)
    assert (mt.gen(3000, host=True) == want).all()
    mt.close()


def test_long_rows_sampled(shv, orc, params):
    """200 streams x 2^20 u32 (800 MB): rows 0, 99, 199 in full."""
    mt = Mt(shv, params, 12345, 0, 200)
    m = 1 << 20
    got = mt.gen(m)
    rows = [0, 99, 199]
    assert (got[rows] == mt.ref(orc, m, streams=rows, offset=0)).all()
    # the state after the call continues exactly
    want = mt.ref(orc, 1000, streams=rows)
    assert (mt.gen(1000)[rows] == want).all()
    mt.close()


def test_mc_counts(shv, orc, params):
    mt = Mt(shv, params, 2026, 0, 200)
    mt.gen(11)  # odd offset: samples pair draws from the call start (R9)
    samples = 20000
    hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    counts = torch.zeros(200, dtype=torch.int64, device="cuda")
    shv.shv_mc_pi_ex(mt.h, samples, hits, counts)
    torch.cuda.synchronize()
    tot, want = orc.mc_count(W.MTGP32, W.mtgp32_seed_words(2026, params), 200, samples, offset=11)
    assert int(hits.item()) == tot
    assert (counts.cpu().numpy() == np.asarray(want)).all()
    mt.offset = 11 + 2 * samples
    want = mt.ref(orc, 100)
    assert (mt.gen(100) == want).all()
    mt.close()


def test_errors(shv, params):
    dev = torch.cuda.current_device()
    with pytest.raises(shv.ShvError) as e:
        shv.shv_streams_create_mtgp32(params, 1, 150, 51, None, 0, dev, None)
    assert e.value.status == shv.SHV_ERR_INSUFFICIENT_STREAMS
    with pytest.raises(shv.ShvError) as e:
        shv.shv_streams_create_mtgp32([], 1, 0, 1, None, 0, dev, None)
    assert e.value.status == shv.SHV_ERR_MISSING_PARAMETERS
    bad = [list(params[0])]
    bad[0][0] = 350
    with pytest.raises(shv.ShvError) as e:
        shv.shv_streams_create_mtgp32(bad, 1, 0, 1, None, 0, dev, None)
    assert e.value.status == shv.SHV_ERR_INVALID_ARGUMENT
    with pytest.raises(shv.ShvError) as e:
        shv.shv_streams_create_ex(shv.SHV_GEN_MTGP32, [1], 0, 1, 0, None, 0, dev, None)
    assert e.value.status == shv.SHV_ERR_MISSING_PARAMETERS
    with pytest.raises(shv.ShvError) as e:
        shv.shv_streams_create_leapfrog(shv.SHV_GEN_MTGP32, [1], 2, 0, 2, None, 0, dev, None)
    assert e.value.status == shv.SHV_ERR_UNSUPPORTED
    h = shv.shv_streams_create_mtgp32(params, 1, 0, 2, None, 0, dev, None)
    with pytest.raises(shv.ShvError) as e:
        shv.shv_get_device_view(h)
    assert e.value.status == shv.SHV_ERR_UNSUPPORTED
    with pytest.raises(shv.ShvError) as e:
        shv.shv_mc_pi(h, 0, torch.zeros(1, dtype=torch.int64, device="cuda"))
    assert e.value.status == shv.SHV_ERR_EMPTY_EXPERIMENT
    shv.shv_streams_destroy(h)
    assert shv.shv_state_bytes(shv.SHV_GEN_MTGP32, 3) == 3 * 1408


def test_jump_is_ordered_on_the_callers_stream(shv, orc, params):
    """Create on stream A, jump on stream B, generate on stream C (SURVEY
    8(b): every call is stream-ordered on its cuda_stream; the caller orders
    the streams with events). The stateful advance must run on B."""
    sa, sb, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(sa):
        h = shv.shv_streams_create_mtgp32(params, 5, 17, 32, None, 0, torch.cuda.current_device(), sa)
    sb.wait_stream(sa)
    shv.shv_jump(h, shv.SHV_JUMP_DRAWS, 3333, sb)
    sc.wait_stream(sb)
    out = torch.empty(32 * 700, dtype=torch.int32, device="cuda")
    shv.shv_generate_u32(h, out, 700, sc)
    sc.synchronize()
    want = orc.generate(W.MTGP32, W.mtgp32_seed_words(5, params), 32, 700, first=17, offset=3333)
    assert (out.cpu().numpy().view(np.uint32).reshape(32, 700) == want).all()
    shv.shv_streams_destroy(h)
