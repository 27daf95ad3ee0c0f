"""Projection kernels (csrc/project.cu) and the projected-SGD driver vs the oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def psgd():
    from paper_2404_11631_b200 import psgd as m
    return m


@pytest.mark.parametrize("d,scale,weighted", [(1, 3.0, False), (10, 0.05, False), (1000, 1.0, False),
                                              (20000, 0.01, False), (1003, 30.0, True),
                                              (10000, 50.0, True)])
def test_project_budget_vs_oracle(psgd, d, scale, weighted):
    rng = np.random.default_rng(d)
    y = rng.standard_normal(d) * scale
    c = rng.uniform(0.5, 2.0, d) if weighted else None
    budget = 0.5 * d if weighted else 1.0
    got = psgd.project_budget(y, c, budget).cpu().numpy()
    want = orc.project_budget(y, c, budget)
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
    cc = np.ones(d) if c is None else c
    assert got.min() >= 0.0 and cc @ got <= budget * (1 + 1e-12)


def test_project_feasible_is_identity_and_box(psgd):
    y = np.array([0.1, 0.2, 0.0, 0.3])
    assert np.array_equal(psgd.project_budget(y).cpu().numpy(), y)
    z = psgd.project_box(np.array([-2.0, 0.5, 9.0]), 0.0, 1.0).cpu().numpy()
    assert np.array_equal(z, [0.0, 0.5, 1.0])


def test_project_nan_raises(psgd):
    from paper_2404_11631_b200.errors import InvalidGradient
    with pytest.raises(InvalidGradient):
        psgd.project_budget(np.array([1.0, np.nan]))


@pytest.mark.parametrize("fused", [False, True])
def test_psgd_meanvar_vs_oracle(psgd, fused):
    import paper_2404_11631_b200 as p
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    b = p.make_backend("cuda")
    task = gen_meanvar_instance(200, p.RngStream(42, 0))
    rec = psgd.psgd_run(MeanVarProblem(task, b, fused=fused),
                        psgd.PsgdConfig(2, 10, 3000, p.RngStream(42, 2), step0=0.5), b)
    mu, sigma = orc.gen_meanvar_instance(200, orc.Stream(42, 0))
    objs, w = orc.psgd_run_meanvar(mu, sigma, 2, 10, 3000, orc.Stream(42, 2), step0=0.5)
    np.testing.assert_allclose(rec.objectives, objs, rtol=1e-8)
    assert np.linalg.norm(rec.final_iterate - w) <= 1e-8 * max(np.linalg.norm(w), 1e-12)
