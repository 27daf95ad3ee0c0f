"""Multi-PRNG kernels (csrc/prng.cu) vs the oracle / numpy, bit for bit."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def prng():
    from paper_2404_11631_b200 import prng as m
    return m


@pytest.mark.parametrize("ctr,key,n", [([0, 0, 0, 0], [0, 0], 1000),
                                       ([0xfffffff0, 0xffffffff, 0xffffffff, 7], [5, 9], 77),
                                       ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                                        [0xa4093822, 0x299f31d0], 1)])
def test_philox4x32_vs_oracle(prng, ctr, key, n):
    got = prng.philox4x32(key, ctr, n).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, orc.philox4x32(ctr, key, n))   # incl. 128-bit counter carry


@pytest.mark.parametrize("n_streams,n", [(1, 5), (37, 100), (300, 33)])
def test_sfc64_streams_vs_numpy(prng, n_streams, n):
    g = prng.Sfc64Streams.from_seed(123, n_streams)
    a = g.raw(n).cpu().numpy().view(np.uint64)
    b = g.random(n).cpu().numpy()                            # continuation
    kids = np.random.SeedSequence(123).spawn(n_streams)
    for k in range(n_streams):
        bg = np.random.SFC64(kids[k])
        assert np.array_equal(a[k], bg.random_raw(n))
        w = bg.random_raw(n)
        assert np.array_equal(b[k], (w >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
        assert np.array_equal(g.host_state()[k], bg.state["state"]["state"])


def test_xoshiro_streams_vs_oracle(prng):
    g = prng.Xoshiro256ppStreams.from_state([1, 2, 3, 4], 40)
    st0 = g.host_state().copy()
    a = g.raw(70).cpu().numpy().view(np.uint64)
    assert list(a[0][:3]) == [41943041, 58720359, 3588806011781223]
    for k in range(40):
        want, st = orc.xoshiro256pp(st0[k], 70)
        assert np.array_equal(a[k], want)
        assert np.array_equal(g.host_state()[k], st)
    assert np.array_equal(st0[1], orc.xoshiro256pp_jump(st0[0]))
