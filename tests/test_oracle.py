"""Pin the CPU oracle to golden vectors produced by the real reference.

Every comparison is bitwise (np.array_equal / ==): the oracle restates the
reference's arithmetic operation for operation.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.conftest import counter_of


def test_philox_known_answer(golden):
    g = golden("rng")
    # Random123 KAT for philox4x64_10(ctr=0, key=0) -- also what numpy emits.
    kat = [0x16554D9ECA36314C, 0xDB20FE9D672D0FDC, 0xD7E772CEE186176B, 0x7E68B68AEC7BA23B]
    assert orc.philox_block([0, 0, 0, 0], [0, 0]) == kat
    assert [int(v) for v in g["kat_zero"]] == kat


@pytest.mark.parametrize("i", range(6))
def test_uniform01_bitwise(golden, i):
    g = golden("rng")
    seed, sid = (int(v) for v in g[f"u{i}_meta"])
    s = orc.Stream(seed, sid, counter_of(g[f"u{i}_ctr"]))
    u = orc.uniform01(s, g[f"u{i}"].size)
    assert np.array_equal(u, g[f"u{i}"])
    assert s.counter == counter_of(g[f"u{i}_after"])


@pytest.mark.parametrize("i", range(4))
def test_standard_normal_bitwise(golden, i):
    g = golden("rng")
    seed, sid = (int(v) for v in g[f"z{i}_meta"])
    s = orc.Stream(seed, sid, counter_of(g[f"z{i}_ctr"]))
    z = orc.standard_normal(s, g[f"z{i}"].size)
    assert np.array_equal(z, g[f"z{i}"])
    assert s.counter == counter_of(g[f"z{i}_after"])


def test_fixed_tree_reductions(golden):
    g = golden("tree")
    for n in (1, 2, 4095, 4096, 4097, 10_000, 3 * 4096 + 1):
        x, y = g[f"x_{n}"], g[f"y_{n}"]
        for chunk in (4096, 3, 64):
            want = g[f"dot_{n}_{chunk}"]
            assert orc.dot(x, y, chunk) == want[0]
            assert orc.vec_sum(x, chunk) == want[1]
    for (r, c) in ((9, 5000), (37, 11), (5000, 13), (4097, 3)):
        a = g[f"A_{r}x{c}"]
        for chunk in (4096, 7):
            assert np.array_equal(orc.matvec(a, g[f"xv_{r}x{c}"], chunk), g[f"mv_{r}x{c}_{chunk}"])
            assert np.array_equal(orc.matvec_t(a, g[f"xt_{r}x{c}"], chunk),
                                  g[f"mvt_{r}x{c}_{chunk}"])


def test_map_kernels(golden):
    g = golden("tree")
    t = g["map_t"]
    assert np.array_equal(orc.sigmoid(t), g["sigmoid"])
    assert np.array_equal(orc.exp(np.clip(t, -700, 700)), g["exp"])
    out = np.empty(t.size)
    orc.lib().orc_logistic_loss_terms(orc._p(t), orc._p(g["loss_z"]), orc._p(out), t.size)
    assert np.array_equal(out, g["loss_terms"])


def test_meanvar(golden):
    g = golden("meanvar")
    s = orc.Stream(42, 2)
    x = orc.sample_returns_diag(g["mu"], g["sigma"], 50, s)
    assert np.array_equal(x, g["X"])
    assert s.counter == counter_of(g["after"])
    for chunk in (4096, 16):
        mean, xc = orc.build_sample_set(x, chunk)
        assert np.array_equal(mean, g[f"mean_{chunk}"])
        assert np.array_equal(xc, g[f"Xc_{chunk}"])
        assert np.array_equal(orc.mv_gradient(g["w"], mean, xc, chunk), g[f"grad_{chunk}"])
        assert orc.mv_objective(g["w"], mean, xc, chunk) == g[f"obj_{chunk}"][0]


@pytest.mark.parametrize("tag", ["a", "b"])
def test_meanvar_fw_trace(golden, tag):
    g = golden("meanvar")
    d, epochs, m_inner, n, chunk = (int(v) for v in g[f"fw{tag}_cfg"])
    mu, sigma = orc.gen_meanvar_instance(d, orc.Stream(42, 0))
    objs, w = orc.fw_run_meanvar(mu, sigma, epochs, m_inner, n, orc.Stream(42, 2), chunk)
    assert np.array_equal(objs, g[f"fw{tag}_obj"])
    assert np.array_equal(w, g[f"fw{tag}_w"])


def test_newsvendor(golden):
    g = golden("newsvendor")
    s = orc.Stream(42, 2)
    dem = orc.sample_demands(g["demand_mean"], g["demand_std"], 301, s)
    assert np.array_equal(dem, g["demands"])
    assert s.counter == counter_of(g["after"])
    k, h, v = g["unit_cost"], g["holding_cost"], g["selling_value"]
    assert np.array_equal(orc.nv_gradient_hat(g["xq"], dem, k, h, v), g["grad"])
    assert orc.nv_objective_exact(g["xq"], g["demand_mean"], g["demand_std"], k, h, v) == g["obj"][0]


@pytest.mark.parametrize("tag", ["a", "b"])
def test_newsvendor_fw_trace(golden, tag):
    g = golden("newsvendor")
    d, epochs, m_inner, n, chunk = (int(v) for v in g[f"fw{tag}_cfg"])
    task = orc.gen_newsvendor_instance(d, orc.Stream(42, 0))
    objs, x = orc.fw_run_newsvendor(task, epochs, m_inner, n, orc.Stream(42, 2), chunk)
    assert np.array_equal(objs, g[f"fw{tag}_obj"])
    assert np.array_equal(x, g[f"fw{tag}_x"])


def test_logistic(golden):
    g = golden("logistic")
    s = orc.Stream(42, 0)
    x, z, w_true = orc.synth_classification(12, s)
    assert np.array_equal(x, g["X"]) and np.array_equal(z, g["z"])
    assert np.array_equal(w_true, g["w_true"])
    assert s.counter == counter_of(g["after"])
    w, v, idx = g["w"], g["v"], g["idx"]
    assert np.array_equal(orc.sample_indices(x.shape[0], 50, orc.Stream(42, 2)), idx)
    assert orc.logistic_loss(w, x, z) == g["loss_full"][0]
    assert orc.logistic_loss(w, x, z, idx) == g["loss_idx"][0]
    assert np.array_equal(orc.logistic_gradient(w, x, z), g["grad_full"])
    assert np.array_equal(orc.logistic_gradient(w, x, z, idx), g["grad_idx"])
    assert np.array_equal(orc.logistic_hvp(w, v, x, z), g["hvp_full"])
    assert np.array_equal(orc.logistic_hvp(w, v, x, z, idx), g["hvp_idx"])
    assert np.array_equal(orc.sample_indices(1000, 400, orc.Stream(10, 0)), g["si_a"])
    assert np.array_equal(orc.sample_indices(10, 10, orc.Stream(9, 0)), g["si_b"])
    pairs = list(zip(g["hu_s"], g["hu_y"], g["hu_curv"]))
    assert np.array_equal(orc.hessian_update(pairs), g["hu_H"])


def test_sqn_trace(golden):
    g = golden("logistic")
    x, z, _ = orc.synth_classification(10, orc.Stream(42, 0))
    objs, w = orc.sqn_run(x, z, pair_every=10, memory=25, beta=2.0, grad_batch=50,
                          hess_batch=100, iterations=60, stream=orc.Stream(42, 2))
    assert np.array_equal(objs, g["sqn_obj"])
    assert np.array_equal(w, g["sqn_w"])


def test_multi_prng_oracle_known_answers():
    """Published known answers for the multi-PRNG restatements (oracle/prng.c)."""
    kat = [([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
           ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
           ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
            [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1])]
    for ctr, key, want in kat:  # Random123 kat_vectors, philox4x32 10 rounds
        assert list(orc.philox4x32(ctr, key, 1)) == want
    out, _ = orc.xoshiro256pp([1, 2, 3, 4], 3)  # xoshiro256plusplus.c from s = {1,2,3,4}
    assert list(out) == [41943041, 58720359, 3588806011781223]
    bg = np.random.SFC64(2024)
    st = bg.state["state"]["state"].copy()
    out, st2 = orc.sfc64(st, 1000)
    assert np.array_equal(out, bg.random_raw(1000))
    assert np.array_equal(st2, bg.state["state"]["state"])


def test_xoshiro_stream_states_host():
    """The library's host stream setup (jump^k) equals the oracle's jump()."""
    from paper_2404_11631_b200.prng import Xoshiro256ppStreams
    import ctypes
    from paper_2404_11631_b200 import _lib
    seed = [0x9E3779B97F4A7C15, 7, 11, 13]
    out = np.empty((3, 4), dtype=np.uint64)
    s = (ctypes.c_uint64 * 4)(*seed)
    _lib.check(_lib.load(require_device=False).simopt_xoshiro256pp_streams(s, 3, out.ctypes.data))
    want = np.array(seed, dtype=np.uint64)
    for k in range(3):
        assert np.array_equal(out[k], want)
        want = orc.xoshiro256pp_jump(want)
    assert Xoshiro256ppStreams is not None


@pytest.mark.parametrize("i", range(7))
def test_lmo_general_golden(golden, i):
    """oracle.lmo_general against the reference's lmo_general (lmo.py:92-160) vertices."""
    g = golden("polytope")
    s = orc.lmo_general(g[f"lp{i}_g"], g[f"lp{i}_A"], g[f"lp{i}_C"])
    assert np.array_equal(s, g[f"lp{i}_s"])


def test_newsvendor_polytope_fw_trace(golden):
    g = golden("polytope")
    task = {"mu": g["fw_demand_mean"], "sigma": g["fw_demand_std"], "k": g["fw_unit_cost"],
            "h": g["fw_holding_cost"], "v": g["fw_selling_value"]}
    objs, x = orc.fw_run_newsvendor_polytope(task, g["fw_A"], g["fw_C"], 2, 5, 400, orc.Stream(42, 2))
    assert np.array_equal(objs, g["fw_obj"])
    assert np.array_equal(x, g["fw_x"])
