"""GPU parity for the second-order drivers (BASELINE configs[2] / [4]) and the DMMA Hessian."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2404_11631_b200 as p
    return p


def _data(pkg, d, n, seed=42):
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.tasks import LogisticTask
    data = synth_classification(d, pkg.RngStream(seed, 0), n_rows=n)
    return LogisticTask(data), data.features.cpu().numpy(), data.labels.cpu().numpy()


def test_newton_cg_bitwise_vs_oracle(pkg):
    from paper_2404_11631_b200.newton import newton_cg
    task, x, z = _data(pkg, 50, 6000)
    rec = newton_cg(task, 4, 10, pkg.make_backend("cuda"), fused=False)
    objs, w = orc.newton_cg(x, z, iterations=4, cg_iters=10)
    assert np.array_equal(rec.objectives, objs)
    assert np.array_equal(rec.final_iterate, w)


@pytest.mark.parametrize("d,n", [(64, 5000), (200, 3001), (13, 777)])
def test_xtdx_dmma_vs_oracle(pkg, d, n):
    from paper_2404_11631_b200.newton import logistic_hessian_device
    task, x, z = _data(pkg, d, n, seed=5)
    rng = np.random.default_rng(d)
    w = rng.standard_normal(d) * 0.2
    want = orc.logistic_hessian_explicit(w, x, z)
    c = orc.sigmoid(orc.matvec(x, w))
    dw = torch.from_numpy(c * (1 - c)).cuda()
    got = logistic_hessian_device(task.data, dw).cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-15)
    assert np.array_equal(got, got.T)


def test_newton_explicit_vs_oracle(pkg):
    from paper_2404_11631_b200.newton import newton_explicit
    task, x, z = _data(pkg, 64, 8000, seed=9)
    rec = newton_explicit(task, 3, 20, pkg.make_backend("cuda"), fused=False)
    objs, w = orc.newton_explicit(x, z, iterations=3, cg_iters=20)
    np.testing.assert_allclose(rec.objectives, objs, rtol=1e-8)
    np.testing.assert_allclose(rec.final_iterate, w, rtol=1e-8, atol=1e-10)
