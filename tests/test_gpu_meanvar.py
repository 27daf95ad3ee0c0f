"""GPU parity for the mean-variance path: sample set, gradient/objective, FW traces (bitwise)."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2404_11631_b200 as p
    return p


def test_sample_set_gradient_objective_golden(pkg, golden):
    from paper_2404_11631_b200.tasks import build_sample_set, mv_gradient, mv_objective
    g = golden("meanvar")
    for chunk in (4096, 16):
        b = pkg.make_backend("cuda", chunk_size=chunk)
        ss = build_sample_set(g["X"], b)
        assert np.array_equal(ss.mean.cpu().numpy(), g[f"mean_{chunk}"])
        assert np.array_equal(ss.centered.cpu().numpy(), g[f"Xc_{chunk}"])
        assert np.array_equal(mv_gradient(g["w"], ss, b), g[f"grad_{chunk}"])
        assert mv_objective(g["w"], ss, b) == g[f"obj_{chunk}"][0]


@pytest.mark.parametrize("tag", ["a", "b"])
def test_fw_trace_golden(pkg, golden, tag):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    g = golden("meanvar")
    d, epochs, m_inner, n, chunk = (int(v) for v in g[f"fw{tag}_cfg"])
    b = pkg.make_backend("cuda", chunk_size=chunk)
    task = gen_meanvar_instance(d, pkg.RngStream(42, 0))
    rec = fw_run(MeanVarProblem(task, b), FwConfig(epochs, m_inner, n, pkg.RngStream(42, 2)), b)
    assert np.array_equal(rec.objectives, g[f"fw{tag}_obj"])
    assert np.array_equal(rec.final_iterate, g[f"fw{tag}_w"])


@pytest.mark.parametrize("d,n,chunk", [(1000, 10_000, 4096), (300, 5000, 256)])
def test_fw_trace_vs_oracle(pkg, d, n, chunk):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    K, M = 2, 25
    b = pkg.make_backend("cuda", chunk_size=chunk)
    task = gen_meanvar_instance(d, pkg.RngStream(42, 0))
    rec = fw_run(MeanVarProblem(task, b), FwConfig(K, M, n, pkg.RngStream(42, 2)), b)
    mu, sigma = orc.gen_meanvar_instance(d, orc.Stream(42, 0))
    objs, w = orc.fw_run_meanvar(mu, sigma, K, M, n, orc.Stream(42, 2), chunk)
    assert np.array_equal(rec.objectives, objs)
    assert np.array_equal(rec.final_iterate, w)
