"""Single-pass fused kernels (csrc/fused.cu) against fp64 numpy and the oracle.

Tolerances (north star): gradients within 1e-10 relative (we assert 1e-12 on the
kernel outputs), trajectories within 1e-8 relative after a fixed budget.
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
    a, b = np.asarray(a, float), np.asarray(b, float)
    den = max(np.linalg.norm(b), 1e-300)
    return np.linalg.norm(a - b) / den


# d covers every cluster width: 1 (C=1), 2500 (C=2), 8192 (C=4), 20000 (C=8), odd d (scalar loads)
@pytest.mark.parametrize("n,d", [(1000, 1), (777, 7), (3001, 1000), (1200, 2500), (300, 8192),
                                 (97, 20000), (5, 999), (1, 64)])
def test_fused_modes_vs_numpy(pkg, n, d):
    from paper_2404_11631_b200.fused import LR_GRAD, LR_HVP, MV, fused_rows
    rng = np.random.default_rng(n * 31 + d)
    x = rng.standard_normal((n, d))
    v = rng.standard_normal(d) * 0.1
    mean = rng.standard_normal(d) * 0.01
    z = (rng.random(n) < 0.5).astype(float)
    dw = rng.random(n) * 0.25
    X, V, Mn, Z, DW = (torch.from_numpy(a).cuda() for a in (x, v, mean, z, dw))
    g, sc = torch.empty(d, dtype=torch.float64, device="cuda"), torch.empty(1, dtype=torch.float64, device="cuda")
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    # MV: g = (Xc^T Xc v) * s - mean, scalar = |Xc v|^2
    s = 1.0 / max(n - 1, 1)
    fused_rows(MV, X, V, center=Mn, col_scale=s, col_out=g, scalar_out=sc, t_out=t)
    xc = x - mean
    q = xc @ v
    assert _rel(t.cpu().numpy(), q) < 1e-13
    assert _rel(g.cpu().numpy(), (xc.T @ q) * s - mean) < 1e-12
    assert abs(sc.item() - q @ q) <= 1e-12 * abs(q @ q)
    # LR_GRAD
    dwo = torch.empty(n, dtype=torch.float64, device="cuda")
    fused_rows(LR_GRAD, X, V, rowaux=Z, col_scale=1.0 / n, col_out=g, scalar_out=sc, dw_out=dwo)
    tt = x @ v
    c = orc.sigmoid(tt)
    assert _rel(g.cpu().numpy(), (x.T @ (c - z)) * (1.0 / n)) < 1e-12
    np.testing.assert_allclose(dwo.cpu().numpy(), c * (1 - c), rtol=1e-12, atol=1e-15)
    loss = np.where(tt >= 0, np.log1p(np.exp(-tt)) + (1 - z) * tt, np.log1p(np.exp(tt)) - z * tt)
    assert abs(sc.item() - loss.sum()) <= 1e-12 * loss.sum()
    # LR_HVP
    fused_rows(LR_HVP, X, V, rowaux=DW, col_scale=1.0 / n, col_out=g)
    assert _rel(g.cpu().numpy(), (x.T @ (dw * tt)) * (1.0 / n)) < 1e-12
    # row pass only
    sc.fill_(-1.0)
    fused_rows(MV, X, V, center=Mn, scalar_out=sc, accumulate=False)
    assert abs(sc.item() - q @ q) <= 1e-12 * abs(q @ q)


def test_fused_deterministic(pkg):
    from paper_2404_11631_b200.fused import MV, fused_rows
    rng = np.random.default_rng(3)
    X = torch.from_numpy(rng.standard_normal((20000, 300))).cuda()
    V = torch.from_numpy(rng.standard_normal(300)).cuda()
    M = torch.zeros(300, dtype=torch.float64, device="cuda")
    outs = []
    for _ in range(3):
        g = torch.empty(300, dtype=torch.float64, device="cuda")
        fused_rows(MV, X, V, center=M, col_out=g)
        outs.append(g.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_fused_empty_and_errors(pkg):
    from paper_2404_11631_b200.errors import ConfigurationError
    from paper_2404_11631_b200.fused import LR_HVP, MV, fused_rows
    X = torch.empty(0, 5, dtype=torch.float64, device="cuda")
    V = torch.ones(5, dtype=torch.float64, device="cuda")
    M = torch.arange(5, dtype=torch.float64, device="cuda")
    g = torch.full((5,), 7.0, dtype=torch.float64, device="cuda")
    sc = torch.full((1,), 7.0, dtype=torch.float64, device="cuda")
    fused_rows(MV, X, V, center=M, col_out=g, scalar_out=sc)
    assert np.array_equal(g.cpu().numpy(), -np.arange(5.0)) and sc.item() == 0.0
    with pytest.raises(ConfigurationError):
        fused_rows(LR_HVP, X, V, col_out=g)            # row weights missing
    with pytest.raises(ConfigurationError):
        fused_rows(7, X, V, center=M, col_out=g)       # unknown mode


def test_newton_cg_fused_vs_oracle(pkg):
    from paper_2404_11631_b200.newton import newton_cg
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.tasks import LogisticTask
    data = synth_classification(50, pkg.RngStream(42, 0), n_rows=6000)
    rec = newton_cg(LogisticTask(data), 4, 10, pkg.make_backend("cuda"), fused=True)
    objs, w = orc.newton_cg(data.features.cpu().numpy(), data.labels.cpu().numpy(),
                            iterations=4, cg_iters=10)
    np.testing.assert_allclose(rec.objectives, objs, rtol=1e-8)
    assert _rel(rec.final_iterate, w) < 1e-8


@pytest.mark.parametrize("d,n", [(1000, 10_000), (300, 5000), (2500, 3000)])
def test_meanvar_fw_fused_vs_oracle(pkg, d, n):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    K, M = 3, 25
    b = pkg.make_backend("cuda")
    task = gen_meanvar_instance(d, pkg.RngStream(42, 0))
    rec = fw_run(MeanVarProblem(task, b, fused=True), FwConfig(K, M, n, pkg.RngStream(42, 2)), b)
    mu, sigma = orc.gen_meanvar_instance(d, orc.Stream(42, 0))
    objs, w = orc.fw_run_meanvar(mu, sigma, K, M, n, orc.Stream(42, 2))
    np.testing.assert_allclose(rec.objectives, objs, rtol=1e-8)
    assert _rel(rec.final_iterate, w) < 1e-8


@pytest.mark.parametrize("d,n", [(1000, 10_000), (513, 2001), (2048, 1500), (2, 50)])
def test_meanvar_persistent_epoch_vs_launch_sequence(pkg, d, n, monkeypatch):
    """The one-launch fused epoch (simopt_mv_fw_epoch, cooperative grid) against the launch
    sequence it replaces (fused pass + finish + tail per step, CUDA graphs) and the oracle:
    same trajectory to 1e-10, oracle to 1e-8 (odd d: scalar loads; d = 2048: K = 4)."""
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    K, M = 3, 25
    b = pkg.make_backend("cuda")
    task = gen_meanvar_instance(d, pkg.RngStream(42, 0))
    recs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SIMOPT_MV_PERSISTENT", flag)
        recs.append(fw_run(MeanVarProblem(task, b, fused=True), FwConfig(K, M, n, pkg.RngStream(42, 2)), b))
    np.testing.assert_allclose(recs[0].objectives, recs[1].objectives, rtol=1e-10)
    assert _rel(recs[0].final_iterate, recs[1].final_iterate) < 1e-10
    assert np.all(np.diff(recs[0].elapsed_ns) >= 0)
    mu, sigma = orc.gen_meanvar_instance(d, orc.Stream(42, 0))
    objs, w = orc.fw_run_meanvar(mu, sigma, K, M, n, orc.Stream(42, 2))
    np.testing.assert_allclose(recs[0].objectives, objs, rtol=1e-8)
    assert _rel(recs[0].final_iterate, w) < 1e-8
