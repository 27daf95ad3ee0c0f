"""The reference's kernel contracts (sobench tests/test_backend.py:1-230) on the "cuda" backend.

Each case restates a reference test with make_backend("cuda") in place of the
sequential/parallel backends; bit-identity between backends becomes bit-identity
with the fixed-tree oracle (a pure-Python restatement as in test_backend.py:23-37,
and oracle/ for the large sizes).  Plus the boundary conventions of SURVEY 8(b):
empty inputs, list/int coercion, inputs never mutated, reentrancy from threads.
"""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2404_11631_b200 as p
    return p


@pytest.fixture(scope="module")
def cuda(pkg):
    return pkg.make_backend("cuda")


def tree_dot_oracle(x, y, chunk=4096):
    """The fixed reduction tree, pure Python (test_backend.py:23-37)."""
    n = len(x)
    partials = []
    for lo in range(0, n, chunk):
        s = 0.0
        for i in range(lo, min(lo + chunk, n)):
            s += x[i] * y[i]
        partials.append(s)
    while len(partials) > 1:
        folded = [partials[2 * i] + partials[2 * i + 1] for i in range(len(partials) // 2)]
        if len(partials) % 2:
            folded.append(partials[-1])
        partials = folded
    return partials[0] if partials else 0.0


# --- dot (test_backend.py:40-92) -----------------------------------------------------------
def test_dot_direct_arithmetic(cuda):
    assert cuda.dot([1.0, 2.0], [3.0, 4.0]) == 11.0
    assert cuda.dot([1, 2], [3, 4]) == 11.0          # integer lists coerced to float64


def test_dot_zero_and_empty(cuda):
    y = np.random.default_rng(0).standard_normal(17)
    assert cuda.dot(np.zeros(17), y) == 0.0
    assert cuda.dot(np.zeros(0), np.zeros(0)) == 0.0  # no partials: 0.0
    assert cuda.vec_sum(np.zeros(0)) == 0.0


@pytest.mark.parametrize("n", [1, 2, 4095, 4096, 4097, 100_000])
def test_dot_matches_tree_oracle_bitwise(cuda, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) * rng.uniform(1e-6, 1e6)
    y = rng.standard_normal(n)
    want = tree_dot_oracle(x, y) if n <= 5000 else orc.dot(x, y)
    assert cuda.dot(x, y) == want


def test_dot_1m_and_symmetry(cuda):
    rng = np.random.default_rng(2)
    x, y = rng.standard_normal(1_000_000), rng.standard_normal(1_000_000)
    assert cuda.dot(x, y) == orc.dot(x, y)
    assert cuda.dot(x, y) == cuda.dot(y, x)


def test_dot_length_mismatch(pkg, cuda):
    with pytest.raises(pkg.DimensionMismatch):
        cuda.dot(np.ones(3), np.ones(4))


@pytest.mark.parametrize("chunk", [1, 3, 64, 1024])
def test_nondefault_chunk_sizes(pkg, chunk):
    rng = np.random.default_rng(4)
    x, y = rng.standard_normal(10_000), rng.standard_normal(10_000)
    b = pkg.make_backend("cuda", chunk_size=chunk)
    assert b.dot(x, y) == tree_dot_oracle(x, y, chunk)


def test_bad_chunk_size(pkg):
    with pytest.raises(pkg.ConfigurationError):
        pkg.make_backend("cuda", chunk_size=0)


def test_vec_sum_matches_dot_with_ones(cuda):
    x = np.random.default_rng(5).standard_normal(30_000)
    assert cuda.vec_sum(x) == cuda.dot(x, np.ones(30_000)) == orc.vec_sum(x)


# --- matvec / matvec_t (test_backend.py:104-165) ------------------------------------------
def test_matvec_small_cases(cuda):
    np.testing.assert_array_equal(cuda.matvec(np.eye(2), [3.0, 5.0]), [3.0, 5.0])
    a = np.array([[1.0, 1.0], [1.0, -1.0]])
    np.testing.assert_array_equal(cuda.matvec(a, [1.0, 1.0]), [2.0, 0.0])
    np.testing.assert_array_equal(cuda.matvec_t(np.eye(2), [3.0, 5.0]), [3.0, 5.0])
    np.testing.assert_array_equal(cuda.matvec_t(np.array([[1.0, 2.0]]), [3.0]), [3.0, 6.0])


def test_matvec_rows_match_dot_bitwise(cuda):
    rng = np.random.default_rng(7)
    a, x = rng.standard_normal((9, 5000)), rng.standard_normal(5000)
    out = cuda.matvec(a, x)
    for i in range(9):
        assert out[i] == cuda.dot(a[i], x)


def test_matvec_linearity(cuda):
    rng = np.random.default_rng(8)
    a = rng.standard_normal((100, 100))
    x, y = rng.standard_normal(100), rng.standard_normal(100)
    alpha, beta = 0.37, -1.42
    lhs = cuda.matvec(a, alpha * x + beta * y)
    rhs = alpha * cuda.matvec(a, x) + beta * cuda.matvec(a, y)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12)


def test_matvec_t_matches_explicit_transpose_bitwise(cuda):
    rng = np.random.default_rng(9)
    a, x = rng.standard_normal((50, 30)), rng.standard_normal(50)
    np.testing.assert_array_equal(cuda.matvec_t(a, x), cuda.matvec(np.ascontiguousarray(a.T), x))


def test_matvec_backends_vs_oracle(cuda):
    rng = np.random.default_rng(6)
    a, x = rng.standard_normal((1000, 200)), rng.standard_normal(200)
    np.testing.assert_array_equal(cuda.matvec(a, x), orc.matvec(a, x))
    a, x = rng.standard_normal((5000, 300)), rng.standard_normal(5000)
    np.testing.assert_array_equal(cuda.matvec_t(a, x), orc.matvec_t(a, x))


def test_matvec_dimension_errors(pkg, cuda):
    with pytest.raises(pkg.DimensionMismatch):
        cuda.matvec(np.eye(3), np.ones(4))
    with pytest.raises(pkg.DimensionMismatch):
        cuda.matvec_t(np.eye(3), np.ones(4))


def test_matvec_non_contiguous_input_not_mutated(cuda):
    rng = np.random.default_rng(21)
    big = rng.standard_normal((40, 60))
    a = big[:, ::2]                                   # non-contiguous view
    x = rng.standard_normal(30)
    a0, x0 = a.copy(), x.copy()
    np.testing.assert_array_equal(cuda.matvec(a, x), orc.matvec(np.ascontiguousarray(a), x))
    assert np.array_equal(a, a0) and np.array_equal(x, x0)


# --- axpy / map_kernel (test_backend.py:167-211) ------------------------------------------
def test_axpy(pkg, cuda):
    np.testing.assert_array_equal(cuda.axpy(0.0, [9.0, 9.0], [1.0, 2.0]), [1.0, 2.0])
    np.testing.assert_array_equal(cuda.axpy(1.0, [1.0, 1.0], [1.0, 2.0]), [2.0, 3.0])
    np.testing.assert_array_equal(cuda.axpy(0.5, [2.0, 0.0], [0.0, 2.0]), [1.0, 2.0])
    with pytest.raises(pkg.DimensionMismatch):
        cuda.axpy(1.0, np.ones(2), np.ones(3))


def test_map_kernels(pkg, cuda):
    np.testing.assert_array_equal(cuda.map_kernel("sigmoid", [0.0]), [0.5])
    out = cuda.map_kernel("sigmoid", [-700.0])
    assert 0.0 < out[0] <= 1e-300 and np.isfinite(out).all()
    t = np.linspace(-40, 40, 1001)
    e = np.exp(-np.abs(t))
    expected = np.where(t >= 0, 1.0 / (1.0 + e), e / (1.0 + e))
    np.testing.assert_allclose(cuda.map_kernel("sigmoid", t), expected, rtol=1e-15)
    np.testing.assert_array_equal(cuda.map_kernel("negate", [1.0, -2.0]), [-1.0, 2.0])
    np.testing.assert_allclose(cuda.map_kernel("exp", [0.0, 1.0]), [1.0, np.e], rtol=1e-15)
    tt = np.random.default_rng(11).standard_normal(200_000) * 10
    np.testing.assert_array_equal(cuda.map_kernel("sigmoid", tt), orc.sigmoid(tt))
    with pytest.raises(pkg.ConfigurationError):
        cuda.map_kernel("tanh", np.ones(3))


# --- reentrancy (test_backend.py:219-228) -------------------------------------------------
def test_concurrent_calls_on_disjoint_data(cuda):
    from concurrent.futures import ThreadPoolExecutor
    rng = np.random.default_rng(12)
    data = [(rng.standard_normal(50_000), rng.standard_normal(50_000)) for _ in range(8)]
    expected = [orc.dot(x, y) for x, y in data]
    with ThreadPoolExecutor(max_workers=4) as pool:
        got = list(pool.map(lambda xy: cuda.dot(*xy), data))
    assert got == expected


def test_reentrant_multi_kernel_ops(cuda):
    """Ops that run as partials + fold (> 64 chunks: dot/vec_sum; matvec with several
    column chunks) from worker threads on one stream: per-thread scratch keeps each
    thread's partials its own (the reference's run_cell runs reps on a ThreadPool)."""
    from concurrent.futures import ThreadPoolExecutor
    rng = np.random.default_rng(13)
    vecs = [(rng.standard_normal(700_000), rng.standard_normal(700_000)) for _ in range(8)]
    mats = [(rng.standard_normal((64, 20_000)), rng.standard_normal(20_000)) for _ in range(8)]
    want_d = [orc.dot(x, y) for x, y in vecs]
    want_s = [orc.vec_sum(x) for x, _ in vecs]
    want_m = [orc.matvec(a, x) for a, x in mats]
    for _ in range(3):
        with ThreadPoolExecutor(max_workers=8) as pool:
            got_d = list(pool.map(lambda xy: cuda.dot(*xy), vecs))
            got_s = list(pool.map(lambda xy: cuda.vec_sum(xy[0]), vecs))
            got_m = list(pool.map(lambda ax: cuda.matvec(*ax), mats))
        assert got_d == want_d and got_s == want_s
        for g, w in zip(got_m, want_m):
            assert np.array_equal(g, w)
