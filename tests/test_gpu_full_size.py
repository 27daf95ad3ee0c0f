"""Parity at BASELINE.json sizes, against golden trajectories the
REAL reference produced (tests/golden/gen_full.py, committed fixtures):

* C2 newsvendor d=10^4, S=10^5, M=25, 3 epochs: final iterate and every recorded
  objective bit for bit (the device loop the bench times).
* C3 logistic Newton-CG d=10^3, N=10^6, k_CG=10: exact tree bit for bit (fp64 and
  bit-packed features), fused single pass within 1e-8.
* C4 mean-variance FW at d=2*10^4, N=2*10^4, one epoch of 25: exact tree bit for bit,
  fused within 1e-8.
* The limb Hessians at n = 2^20 + 12289 samples (two launches per limb pass, so the
  cross-launch accumulation runs) and d = 1024, against DMMA and a CPU oracle block, and
  the precision guard on a confident model (tiny c(1-c) for most samples).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2404_11631_b200 as p
    return p


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def test_c2_full_size_trace(pkg, golden):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    g = golden("full_c2")
    d, S, M, K = (int(v) for v in g["meta"])
    b = pkg.make_backend("cuda")
    rec = fw_run(NewsvendorProblem(gen_newsvendor_instance(d, pkg.RngStream(42, 0)), b),
                 FwConfig(K, M, S, pkg.RngStream(42, 2)), b)
    assert np.array_equal(rec.final_iterate, g["final_iterate"])
    assert np.array_equal(rec.objectives, g["objectives"])


@pytest.fixture(scope="module")
def c3_data(pkg):
    from paper_2404_11631_b200.sampling import synth_classification
    d, N = 1_000, 1_000_000
    dense = synth_classification(d, pkg.RngStream(42, 0), n_rows=N)
    packed = synth_classification(d, pkg.RngStream(42, 0), n_rows=N, packed=True)
    return dense, packed


def test_c3_full_size_instance(c3_data, golden):
    g = golden("full_c3")
    dense, packed = c3_data
    assert float(dense.labels.sum().item()) == float(g["labels_sum"][0])
    assert torch.equal(dense.labels, packed.labels)


@pytest.mark.parametrize("features", ["fp64", "bits"])
def test_c3_full_size_newton_cg(pkg, c3_data, golden, features):
    from paper_2404_11631_b200.newton import newton_cg
    from paper_2404_11631_b200.tasks import LogisticTask
    g = golden("full_c3")
    d, N, iters, kcg = (int(v) for v in g["meta"])
    data = c3_data[0] if features == "fp64" else c3_data[1]
    b = pkg.make_backend("cuda")
    rec = newton_cg(LogisticTask(data), iters, kcg, b, fused=False)   # exact fixed tree
    assert np.array_equal(rec.objectives, g["objectives"])
    assert np.array_equal(rec.final_iterate, g["final_iterate"])
    rec = newton_cg(LogisticTask(data), iters, kcg, b, fused=True)    # one read of X per pass
    np.testing.assert_allclose(rec.objectives, g["objectives"], rtol=1e-8)
    assert _rel(rec.final_iterate, g["final_iterate"]) < 1e-8


def test_c4_full_size_epoch(pkg, golden):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    g = golden("full_c4")
    d, N, M, K = (int(v) for v in g["meta"])
    b = pkg.make_backend("cuda")
    task = gen_meanvar_instance(d, pkg.RngStream(42, 0))
    rec = fw_run(MeanVarProblem(task, b), FwConfig(K, M, N, pkg.RngStream(42, 2)), b)
    assert np.array_equal(rec.objectives, g["objectives"])
    assert np.array_equal(rec.final_iterate, g["final_iterate"])
    rec = fw_run(MeanVarProblem(task, b, fused=True), FwConfig(K, M, N, pkg.RngStream(42, 2)), b)
    np.testing.assert_allclose(rec.objectives, g["objectives"], rtol=1e-8)
    assert _rel(rec.final_iterate, g["final_iterate"]) < 1e-8


@pytest.fixture(scope="module")
def big_bits(pkg):
    from paper_2404_11631_b200.sampling import synth_classification
    n, d = (1 << 20) + 12_289, 1024
    return synth_classification(d, pkg.RngStream(11, 0), n_rows=n, packed=True)


def _block_oracle(data, dw, cols):
    """H[cols][:, cols] on the CPU: (x.T * dw) @ x / n over those columns (the reference
    test's expression, tests/test_tasks.py:297-299), fp64 numpy."""
    x = data.features[:, cols].cpu().numpy()
    return (x.T * dw.cpu().numpy()) @ x / x.shape[0]


@pytest.mark.parametrize("spread", ["moderate", "confident"])
def test_limb_hessian_multi_launch(pkg, big_bits, spread):
    from paper_2404_11631_b200.newton import logistic_hessian_device
    data = big_bits
    n = data.local_rows
    gen = torch.Generator(device="cuda").manual_seed(3)
    if spread == "moderate":    # c(1-c) of an uncertain model: one limb pass
        dw = torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) * 0.25
    else:                        # a confident model: most c(1-c) ~1e-6, a few near 1/4
        t = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen) * 4.0 + 12.0
        c = torch.sigmoid(t)
        dw = c * (1 - c)
    ref = logistic_hessian_device(data, dw, method="dmma")
    cols = np.r_[0:96, 900:1024]
    want = _block_oracle(data, dw, cols)
    np.testing.assert_allclose(ref.cpu().numpy()[np.ix_(cols, cols)], want, rtol=1e-10, atol=0)
    for method in ("tma", "tc", "i8"):
        got = logistic_hessian_device(data, dw, method=method)
        passes = logistic_hessian_device.last_passes
        assert passes == (1 if spread == "moderate" else 3), (method, passes)
        np.testing.assert_allclose(got.cpu().numpy(), ref.cpu().numpy(), rtol=1e-10, atol=0,
                                   err_msg=method)
        np.testing.assert_allclose(got.cpu().numpy()[np.ix_(cols, cols)], want, rtol=1e-10, atol=0,
                                   err_msg=method)
