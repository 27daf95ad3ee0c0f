"""GPU parity: sampling + fixed-tree kernels vs the oracle and the golden vectors (bitwise)."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from tests.conftest import counter_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2404_11631_b200 as p
    return p


@pytest.mark.parametrize("i", range(6))
def test_uniform01_golden(pkg, golden, i):
    g = golden("rng")
    seed, sid = (int(v) for v in g[f"u{i}_meta"])
    s = pkg.RngStream(seed, sid, counter_of(g[f"u{i}_ctr"]) & ((1 << 128) - 1))
    u = pkg.uniform01(s, g[f"u{i}"].size)
    assert np.array_equal(u, g[f"u{i}"])
    assert s.counter == counter_of(g[f"u{i}_after"])


@pytest.mark.parametrize("i", range(4))
def test_standard_normal_golden(pkg, golden, i):
    g = golden("rng")
    seed, sid = (int(v) for v in g[f"z{i}_meta"])
    s = pkg.RngStream(seed, sid, counter_of(g[f"z{i}_ctr"]))
    z = pkg.standard_normal(s, g[f"z{i}"].size)
    assert np.array_equal(z, g[f"z{i}"])
    assert s.counter == counter_of(g[f"z{i}_after"])


@pytest.mark.parametrize("seed,sid,ctr,n", [(42, 1, 0, 3_000_001), (2**64 - 1, 7, 2**64 - 5, 1_000_003),
                                            (3, 2**63, 12345, 4)])
def test_standard_normal_vs_oracle_large(pkg, seed, sid, ctr, n):
    z = pkg.standard_normal(pkg.RngStream(seed, sid, ctr), n)
    want = orc.standard_normal(orc.Stream(seed, sid, ctr), n)
    mism = np.flatnonzero(z.view(np.uint64) != want.view(np.uint64))
    assert mism.size == 0, f"{mism.size} mismatches, first at {mism[:5]}"


def test_normals_1e8_bitwise(pkg):
    """10^8 device normals vs the glibc-backed oracle (the survey's >=1e9 gate is in bench)."""
    n = 100_000_000
    z = pkg.standard_normal_device(pkg.RngStream(42, 2), n)
    want = torch.from_numpy(orc.standard_normal(orc.Stream(42, 2), n)).cuda()
    bad = int((z.view(torch.int64) != want.view(torch.int64)).sum().item())
    assert bad == 0


def test_sample_returns_golden(pkg, golden):
    g = golden("meanvar")
    spec = pkg.GaussianSpec(mean=g["mu"], diag_std=g["sigma"])
    s = pkg.RngStream(42, 2)
    x = pkg.sample_returns(spec, 50, s)
    assert np.array_equal(x, g["X"])
    assert s.counter == counter_of(g["after"])


def test_tree_golden(pkg, golden):
    g = golden("tree")
    for n in (1, 2, 4095, 4096, 4097, 10_000, 3 * 4096 + 1):
        x, y = g[f"x_{n}"], g[f"y_{n}"]
        for chunk in (4096, 3, 64):
            b = pkg.make_backend("cuda", chunk_size=chunk)
            want = g[f"dot_{n}_{chunk}"]
            assert b.dot(x, y) == want[0], (n, chunk)
            assert b.vec_sum(x) == want[1], (n, chunk)
    for (r, c) in ((9, 5000), (37, 11), (5000, 13), (4097, 3)):
        a = g[f"A_{r}x{c}"]
        for chunk in (4096, 7):
            b = pkg.make_backend("cuda", chunk_size=chunk)
            assert np.array_equal(b.matvec(a, g[f"xv_{r}x{c}"]), g[f"mv_{r}x{c}_{chunk}"]), (r, c, chunk)
            assert np.array_equal(b.matvec_t(a, g[f"xt_{r}x{c}"]), g[f"mvt_{r}x{c}_{chunk}"]), (r, c, chunk)


def test_map_kernels_golden(pkg, golden):
    g = golden("tree")
    b = pkg.make_backend("cuda")
    t = g["map_t"]
    assert np.array_equal(b.map_kernel("sigmoid", t), g["sigmoid"])
    assert np.array_equal(b.map_kernel("exp", np.clip(t, -700, 700)), g["exp"])
    assert np.array_equal(b.map_kernel("negate", t), -t)


@pytest.mark.parametrize("rows,cols,chunk", [(10_000, 1000, 4096), (3000, 9000, 4096), (1000, 300, 64),
                                             (70_000, 17, 4096)])
def test_matvec_vs_oracle(pkg, rows, cols, chunk):
    rng = np.random.default_rng(rows + cols)
    a = rng.standard_normal((rows, cols))
    x = rng.standard_normal(cols)
    xt = rng.standard_normal(rows)
    center = rng.standard_normal(cols)
    b = pkg.make_backend("cuda", chunk_size=chunk)
    assert np.array_equal(b.matvec(a, x), orc.matvec(a, x, chunk))
    assert np.array_equal(b.matvec_t(a, xt), orc.matvec_t(a, xt, chunk))
    ad = torch.from_numpy(a).cuda()
    cd = torch.from_numpy(center).cuda()
    got = b.matvec_device(ad, torch.from_numpy(x).cuda(), center=cd).cpu().numpy()
    assert np.array_equal(got, orc.matvec(a - center[None, :], x, chunk))
    got = b.matvec_t_device(ad, torch.from_numpy(xt).cuda(), center=cd).cpu().numpy()
    assert np.array_equal(got, orc.matvec_t(a - center[None, :], xt, chunk))
    idx = rng.choice(rows, size=min(rows, 300), replace=False).astype(np.int64)
    got = b.matvec_device(ad, torch.from_numpy(x).cuda(), rows_idx=torch.from_numpy(idx).cuda()).cpu().numpy()
    assert np.array_equal(got, orc.matvec(a[idx], x, chunk))


def test_dot_large(pkg):
    rng = np.random.default_rng(5)
    x = rng.standard_normal(3_000_001)
    y = rng.standard_normal(3_000_001)
    b = pkg.make_backend("cuda")
    assert b.dot(x, y) == orc.dot(x, y)
    assert b.vec_sum(x) == orc.vec_sum(x)


@pytest.mark.parametrize("n", [0, 1, 1000, 8192, 65536])
def test_dot_fast(pkg, n):
    """simopt_dot_fast: the fused CG's deterministic one-CTA dot -- its own fixed order
    (thread-strided sums, warp xor trees), reproduced here in numpy, and within 1e-13 of
    the exact value."""
    import torch
    from paper_2404_11631_b200 import _lib
    rng = np.random.default_rng(n + 7)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    _lib.call("simopt_dot_fast", _lib.stream_ptr(), _lib.ptr(xd), _lib.ptr(yd), n, _lib.ptr(out))
    got = float(out.item())
    # restatement of the kernel's order
    T = 1024
    s = np.zeros(T)
    for t in range(T):
        acc = 0.0
        for i in range(t, n, T):
            acc += float(x[i] * y[i])
        s[t] = acc

    def xor_tree(v):
        v = v.copy()
        for o in (16, 8, 4, 2, 1):
            v = v + v[np.arange(32) ^ o]
        return v[0]
    w = np.array([xor_tree(s[32 * k:32 * k + 32]) for k in range(32)])
    assert got == xor_tree(w)
    exact = float(np.dot(x.astype(np.longdouble), y.astype(np.longdouble))) if n else 0.0
    assert abs(got - exact) <= 1e-13 * max(1.0, float(np.abs(x * y).sum()))


@pytest.mark.parametrize("rows,cols", [(10_000, 1000), (65, 33), (1, 5), (200, 1)])
def test_col_sums_fast(pkg, rows, cols):
    """simopt_col_sums_fast (the fused mean-variance mean at small N): 256 row groups of
    ceil(rows/256) summed sequentially per column, partials folded in group order."""
    from paper_2404_11631_b200 import _lib
    rng = np.random.default_rng(rows + cols)
    x = rng.standard_normal((rows, cols))
    out = torch.empty(cols, dtype=torch.float64, device="cuda")
    _lib.call("simopt_col_sums_fast", _lib.stream_ptr(), _lib.ptr(torch.from_numpy(x).cuda()), rows, cols,
              _lib.ptr(out))
    R = -(-rows // 256)
    want = np.zeros(cols)
    for g in range(256):
        part = np.zeros(cols)
        for r in range(g * R, min((g + 1) * R, rows)):
            part = part + x[r]
        want = want + part
    assert np.array_equal(out.cpu().numpy(), want)


def test_errors(pkg):
    b = pkg.make_backend("cuda")
    with pytest.raises(pkg.DimensionMismatch):
        b.dot(np.ones(3), np.ones(4))
    with pytest.raises(pkg.DimensionMismatch):
        b.matvec(np.eye(3), np.ones(4))
    with pytest.raises(pkg.ConfigurationError):
        b.map_kernel("tanh", np.ones(3))
    with pytest.raises(pkg.ConfigurationError):
        pkg.make_backend("gpu")
    with pytest.raises(pkg.EmptyRequest):
        pkg.uniform01(pkg.RngStream(1, 0), 0)


def test_philox_floor_words():
    """simopt_philox_floor runs the resample's Philox core: the XOR of every word of blocks
    clo+1 .. clo+n equals numpy's Philox4x64 stream (bench.py's compute_roof measures it)."""
    import numpy as np
    import torch
    from paper_2404_11631_b200 import _lib
    seed, sid, clo, n = 42, 2, 12345, 100_003
    nw = 8 * torch.cuda.get_device_properties(0).multi_processor_count * 256
    out = torch.empty(nw, dtype=torch.int64, device="cuda")
    _lib.call("simopt_philox_floor", _lib.stream_ptr(), seed, sid, clo, n, _lib.ptr(out), nw)
    got = np.bitwise_xor.reduce(out.cpu().numpy().view(np.uint64))
    bg = np.random.Philox(key=np.array([seed, sid], dtype=np.uint64),
                          counter=np.array([clo, 0, 0, 0], dtype=np.uint64))
    want = np.bitwise_xor.reduce(bg.random_raw(4 * n).astype(np.uint64))
    assert got == want
