"""Bit-packed binary features (csrc/bits.cu): generation, exact scores, fused passes,
DMMA Hessian -- against the fp64 layout (bitwise where the arithmetic is identical) and
the oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2404_11631_b200 as p
    return p


@pytest.mark.parametrize("d,n", [(40, 1200), (63, 777), (64, 500), (130, 1000), (1000, 3000)])
def test_packed_synth_equals_dense(pkg, d, n):
    from paper_2404_11631_b200.sampling import synth_classification
    a = synth_classification(d, pkg.RngStream(42, 0), n_rows=n)
    b = synth_classification(d, pkg.RngStream(42, 0), n_rows=n, packed=True)
    assert b.packed and b.n_features == d and b.n_samples == n
    assert torch.equal(a.labels, b.labels) and torch.equal(a.true_weights, b.true_weights)
    assert torch.equal(a.features, b.features)          # device unpack of the bits
    x, z, _ = orc.synth_classification(d, orc.Stream(42, 0), n_rows=n)
    assert np.array_equal(b.labels.cpu().numpy(), z)


@pytest.mark.parametrize("chunk", [4096, 100, 64, 7])
def test_matvec_bits_exact(pkg, chunk):
    from paper_2404_11631_b200 import _lib
    from paper_2404_11631_b200.sampling import synth_classification
    data = synth_classification(300, pkg.RngStream(3, 0), n_rows=2000, packed=True)
    v = torch.from_numpy(np.random.default_rng(1).standard_normal(300)).cuda()
    out = torch.empty(2000, dtype=torch.float64, device="cuda")
    _lib.call("simopt_matvec_bits", _lib.stream_ptr(), _lib.ptr(data.bits), 2000, 300, _lib.ptr(v),
              chunk, _lib.ptr(out))
    want = orc.matvec(data.features.cpu().numpy(), v.cpu().numpy(), chunk)
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("d,n,chunk,gather", [(300, 2000, 4096, True), (1000, 3001, 4096, False),
                                               (1000, 3001, 128, True), (8192, 257, 4096, True),
                                               (70, 9000, 64, False), (5, 40, 4096, True)])
def test_matvec_bits_gather_and_transpose_exact(pkg, d, n, chunk, gather):
    """matvec_bits_idx / matvec_t_bits (slab kernel, row gather, column sums) bitwise equal
    the fixed-tree oracle on the 0/1 matrix, negative zeros and chunk cuts included."""
    from paper_2404_11631_b200 import _lib
    from paper_2404_11631_b200.sampling import synth_classification
    data = synth_classification(d, pkg.RngStream(5, 0), n_rows=n, packed=True)
    rng = np.random.default_rng(d + n)
    v = rng.standard_normal(d)
    v[::7] = -0.0
    if d == 70:
        v[10] = np.inf   # the reference's 0.0 * inf is NaN: every row's dot is NaN or inf
    b = min(n, 777) if gather else n
    idx = rng.choice(n, size=b, replace=False) if gather else None
    x = data.features.cpu().numpy()
    xb = x[idx] if gather else x
    vd = torch.from_numpy(v).cuda()
    idd = torch.from_numpy(idx).cuda() if gather else None
    out = torch.empty(b, dtype=torch.float64, device="cuda")
    _lib.call("simopt_matvec_bits_idx", _lib.stream_ptr(), _lib.ptr(data.bits), n, d, _lib.ptr(idd),
              b, _lib.ptr(vd), chunk, _lib.ptr(out))
    assert np.array_equal(out.cpu().numpy(), orc.matvec(xb, v, chunk), equal_nan=True)
    r = rng.standard_normal(b)
    r[::5] = -0.0
    if d == 70:
        r[3] = -np.inf
    outt = torch.empty(d, dtype=torch.float64, device="cuda")
    _lib.call("simopt_matvec_t_bits", _lib.stream_ptr(), _lib.ptr(data.bits), n, d, _lib.ptr(idd),
              b, _lib.ptr(torch.from_numpy(r).cuda()), chunk, _lib.ptr(outt))
    got, want = outt.cpu().numpy(), orc.matvec_t(xb, r, chunk)
    assert np.array_equal(got, want, equal_nan=True)
    assert np.array_equal(np.signbit(got), np.signbit(want))


@pytest.mark.parametrize("d,n", [(1000, 5000), (8192, 300), (130, 999), (5, 64), (2000, 3001),
                                 (1100, 700), (8192, 20_000)])
def test_fused_bits_vs_dense(pkg, d, n):
    """Nibble-table pass (d <= 1024) and the banded two-sweep pass (d > 1024)."""
    from paper_2404_11631_b200.fused import LR_GRAD, LR_HVP, fused_rows_bits
    from paper_2404_11631_b200.sampling import synth_classification
    data = synth_classification(d, pkg.RngStream(9, 0), n_rows=n, packed=True)
    x = data.features.cpu().numpy()
    z = data.labels.cpu().numpy()
    rng = np.random.default_rng(d)
    w = rng.standard_normal(d) * 0.05
    W = torch.from_numpy(w).cuda()
    g = torch.empty(d, dtype=torch.float64, device="cuda")
    sc = torch.empty(1, dtype=torch.float64, device="cuda")
    dw = torch.empty(n, dtype=torch.float64, device="cuda")
    fused_rows_bits(LR_GRAD, data.bits, d, W, rowaux=data.labels, col_scale=1.0 / n, col_out=g,
                    scalar_out=sc, dw_out=dw)
    t = x @ w
    c = orc.sigmoid(t)
    want = (x.T @ (c - z)) / n
    assert np.linalg.norm(g.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want)
    loss = np.where(t >= 0, np.log1p(np.exp(-t)) + (1 - z) * t, np.log1p(np.exp(t)) - z * t)
    assert abs(sc.item() - loss.sum()) <= 1e-12 * loss.sum()
    np.testing.assert_allclose(dw.cpu().numpy(), c * (1 - c), rtol=1e-12, atol=1e-15)
    v = rng.standard_normal(d)
    fused_rows_bits(LR_HVP, data.bits, d, torch.from_numpy(v).cuda(), rowaux=dw, col_scale=1.0 / n,
                    col_out=g)
    want = (x.T @ ((c * (1 - c)) * (x @ v))) / n
    assert np.linalg.norm(g.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("d,n", [(64, 5000), (200, 3001), (13, 777)])
def test_xtdx_bits_equals_dense(pkg, d, n):
    from paper_2404_11631_b200.newton import logistic_hessian_device
    from paper_2404_11631_b200.sampling import synth_classification
    dense = synth_classification(d, pkg.RngStream(5, 0), n_rows=n)
    packed = synth_classification(d, pkg.RngStream(5, 0), n_rows=n, packed=True)
    dw = torch.rand(n, dtype=torch.float64, device="cuda") * 0.25
    assert torch.equal(logistic_hessian_device(dense, dw), logistic_hessian_device(packed, dw, method="dmma"))


@pytest.mark.parametrize("method", ["i8", "tc", "tma", "pair"])
@pytest.mark.parametrize("d,n", [(128, 4096), (200, 3001), (13, 777), (1000, 2000), (300, 40),
                                 (97, 9000)])
def test_xtdx_i8_vs_oracle(pkg, d, n, method):
    """Integer-tensor-core Hessian (exact limbs of dw rounded to 2^-41) vs the explicit oracle."""
    from paper_2404_11631_b200.newton import logistic_hessian_device
    from paper_2404_11631_b200.sampling import synth_classification
    data = synth_classification(d, pkg.RngStream(5, 0), n_rows=n, packed=True)
    rng = np.random.default_rng(d)
    w = rng.standard_normal(d) * 0.2
    x, z = data.features.cpu().numpy(), data.labels.cpu().numpy()
    want = orc.logistic_hessian_explicit(w, x, z)
    c = orc.sigmoid(orc.matvec(x, w))
    dw = torch.from_numpy(c * (1 - c)).cuda()
    got = logistic_hessian_device(data, dw, method=method).cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-15)
    assert np.array_equal(got, got.T)
    dmma = logistic_hessian_device(data, dw, method="dmma").cpu().numpy()
    np.testing.assert_allclose(got, dmma, rtol=1e-10, atol=1e-15)
    # dw = 1/4 everywhere (w = 0): the largest fixed-point value
    quarter = torch.full((n,), 0.25, dtype=torch.float64, device="cuda")
    np.testing.assert_allclose(logistic_hessian_device(data, quarter, method=method).cpu().numpy(),
                               (x.T @ x) * 0.25 / n, rtol=1e-12)


@pytest.mark.parametrize("d,n", [(1000, 70_000), (256, 5000), (130, 64)])
def test_xtdx_tma_equals_tc(pkg, d, n):
    """TMA-fed and cp.async-fed tcgen05 kernels: the same integer sums, the same bits."""
    from paper_2404_11631_b200.newton import logistic_hessian_device
    from paper_2404_11631_b200.sampling import synth_classification
    data = synth_classification(d, pkg.RngStream(8, 0), n_rows=n, packed=True)
    dw = torch.rand(n, dtype=torch.float64, device="cuda") * 0.25
    ref = logistic_hessian_device(data, dw, method="tc")
    assert torch.equal(logistic_hessian_device(data, dw, method="tma"), ref)
    assert torch.equal(logistic_hessian_device(data, dw, method="pair"), ref)


def test_newton_packed_vs_oracle(pkg):
    from paper_2404_11631_b200.newton import newton_cg, newton_explicit
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.tasks import LogisticTask
    data = synth_classification(50, pkg.RngStream(42, 0), n_rows=6000, packed=True)
    x, z, _ = orc.synth_classification(50, orc.Stream(42, 0), n_rows=6000)
    b = pkg.make_backend("cuda")
    rec = newton_cg(LogisticTask(data), 4, 10, b)                 # fused, bits
    objs, w = orc.newton_cg(x, z, iterations=4, cg_iters=10)
    np.testing.assert_allclose(rec.objectives, objs, rtol=1e-8)
    assert np.linalg.norm(rec.final_iterate - w) <= 1e-8 * np.linalg.norm(w)
    rec = newton_cg(LogisticTask(data), 4, 10, b, fused=False)    # exact tree on unpacked rows
    assert np.array_equal(rec.objectives, objs) and np.array_equal(rec.final_iterate, w)
    rec = newton_explicit(LogisticTask(data), 3, 20, b)
    objs, w = orc.newton_explicit(x, z, iterations=3, cg_iters=20)
    np.testing.assert_allclose(rec.objectives, objs, rtol=1e-8)
    assert np.linalg.norm(rec.final_iterate - w) <= 1e-8 * np.linalg.norm(w)
