"""GPU parity for the classification task: synthetic data, loss/gradient/HVP, BFGS, SQN traces."""
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


@pytest.mark.parametrize("packed", [False, True])
def test_synth_and_logistic_kernels_golden(pkg, packed, golden):
    from paper_2404_11631_b200.sampling import sample_indices, synth_classification
    from paper_2404_11631_b200 import tasks as T
    g = golden("logistic")
    s = pkg.RngStream(42, 0)
    data = synth_classification(12, s, packed=packed)
    assert np.array_equal(data.features.cpu().numpy(), g["X"])
    assert np.array_equal(data.labels.cpu().numpy(), g["z"])
    assert np.array_equal(data.true_weights.cpu().numpy(), g["w_true"])
    assert s.counter == counter_of(g["after"])
    b = pkg.make_backend("cuda")
    w, v, idx = g["w"], g["v"], g["idx"]
    assert np.array_equal(sample_indices(data.n_samples, 50, pkg.RngStream(42, 2)), idx)
    assert T.logistic_loss(w, data, None, b) == g["loss_full"][0]
    assert T.logistic_loss(w, data, idx, b) == g["loss_idx"][0]
    assert np.array_equal(T.logistic_gradient(w, data, None, b), g["grad_full"])
    assert np.array_equal(T.logistic_gradient(w, data, idx, b), g["grad_idx"])
    assert np.array_equal(T.logistic_hvp(w, v, data, None, b), g["hvp_full"])
    assert np.array_equal(T.logistic_hvp(w, v, data, idx, b), g["hvp_idx"])
    assert np.array_equal(sample_indices(1000, 400, pkg.RngStream(10, 0)), g["si_a"])
    assert np.array_equal(sample_indices(10, 10, pkg.RngStream(9, 0)), g["si_b"])


def test_hessian_update_golden(pkg, golden):
    from paper_2404_11631_b200.sqn import CorrectionPair, hessian_update
    g = golden("logistic")
    pairs = [CorrectionPair(s=torch.from_numpy(s).cuda(), y=torch.from_numpy(y).cuda(), curvature=float(c))
             for s, y, c in zip(g["hu_s"], g["hu_y"], g["hu_curv"])]
    h = hessian_update(pairs, 4, 25, pkg.make_backend("cuda"))
    assert np.array_equal(h.cpu().numpy(), g["hu_H"])


@pytest.mark.parametrize("packed", [False, True])
def test_sqn_trace_golden(pkg, packed, golden):
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.sqn import SqnConfig, sqn_run
    from paper_2404_11631_b200.tasks import LogisticTask
    g = golden("logistic")
    b = pkg.make_backend("cuda")
    data = synth_classification(10, pkg.RngStream(42, 0), packed=packed)
    rec = sqn_run(LogisticTask(data), SqnConfig(10, 25, 2.0, 50, 100, 60, pkg.RngStream(42, 2)), b)
    assert np.array_equal(rec.objectives, g["sqn_obj"])
    assert np.array_equal(rec.final_iterate, g["sqn_w"])


@pytest.mark.parametrize("packed,graph", [(False, True), (True, True), (False, False)])
def test_sqn_vs_oracle_larger(pkg, packed, graph):
    """graph=True: the CUDA-graph iteration (SqnGraphRunner); False: the eager engine."""
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.sqn import SqnConfig, sqn_run
    from paper_2404_11631_b200.tasks import LogisticTask
    d, K = 100, 80
    b = pkg.make_backend("cuda")
    data = synth_classification(d, pkg.RngStream(42, 0), packed=packed)
    rec = sqn_run(LogisticTask(data), SqnConfig(10, 25, 2.0, 50, 300, K, pkg.RngStream(42, 2)), b,
                  graph=graph)
    x, z, _ = orc.synth_classification(d, orc.Stream(42, 0))
    objs, w = orc.sqn_run(x, z, pair_every=10, memory=25, beta=2.0, grad_batch=50, hess_batch=300,
                          iterations=K, stream=orc.Stream(42, 2))
    assert np.array_equal(rec.objectives, objs)
    assert np.array_equal(rec.final_iterate, w)


@pytest.mark.parametrize("d,n_rows", [(64, 20_000), (33, 4097)])
def test_synth_generalised_vs_oracle(pkg, d, n_rows):
    from paper_2404_11631_b200.sampling import synth_classification
    s = pkg.RngStream(7, 0)
    data = synth_classification(d, s, n_rows=n_rows)
    os_ = orc.Stream(7, 0)
    x, z, w = orc.synth_classification(d, os_, n_rows=n_rows)
    assert np.array_equal(data.features.cpu().numpy(), x)
    assert np.array_equal(data.labels.cpu().numpy(), z)
    assert s.counter == os_.counter


@pytest.mark.parametrize("packed", [False, True])
def test_full_gradient_hvp_vs_oracle(pkg, packed):
    """Packed: the exact-tree passes read the bits (matvec_bits_idx / matvec_t_bits)."""
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200 import tasks as T
    d, n = 300, 50_000
    data = synth_classification(d, pkg.RngStream(3, 0), n_rows=n, packed=packed)
    x, z = data.features.cpu().numpy(), data.labels.cpu().numpy()
    rng = np.random.default_rng(1)
    w, v = rng.standard_normal(d) * 0.1, rng.standard_normal(d)
    b = pkg.make_backend("cuda")
    assert np.array_equal(T.logistic_gradient(w, data, None, b), orc.logistic_gradient(w, x, z))
    assert np.array_equal(T.logistic_hvp(w, v, data, None, b), orc.logistic_hvp(w, v, x, z))
    assert T.logistic_loss(w, data, None, b) == orc.logistic_loss(w, x, z)


@pytest.mark.parametrize("packed", [False, True])
def test_sqn_graph_equals_eager_with_warnings(pkg, packed):
    """Graph and eager iterations give the same trace, iterate and warnings on a
    configuration with pair iterations every 3 steps and 2-sample HVP batches."""
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.sqn import SqnConfig, sqn_run
    from paper_2404_11631_b200.tasks import LogisticTask
    b = pkg.make_backend("cuda")
    data = synth_classification(24, pkg.RngStream(11, 0), packed=packed)
    recs = [sqn_run(LogisticTask(data), SqnConfig(3, 3, 0.5, 5, 2, 40, pkg.RngStream(11, 2)), b, graph=g)
            for g in (True, False)]
    assert np.array_equal(recs[0].objectives, recs[1].objectives)
    assert np.array_equal(recs[0].final_iterate, recs[1].final_iterate)
    assert recs[0].warnings == recs[1].warnings


def test_sqn_abort_path_graph_equals_eager(pkg):
    """A 1-sample HVP batch eventually yields a pair whose y.y underflows to zero: the
    reference's hessian_update raises DegeneratePair (sqn.py:94-95) and sqn_run turns it
    into RunAborted with the partial trace (sqn.py:186-193).  Both iteration modes must
    stop at the same iteration with the same partial record."""
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.sqn import SqnConfig, sqn_run
    from paper_2404_11631_b200.tasks import LogisticTask
    b = pkg.make_backend("cuda")
    data = synth_classification(24, pkg.RngStream(11, 0))
    parts = []
    for g in (True, False):
        with pytest.raises(pkg.RunAborted) as ei:
            sqn_run(LogisticTask(data), SqnConfig(2, 3, 0.5, 5, 1, 40, pkg.RngStream(11, 2)), b, graph=g)
        assert isinstance(ei.value.__cause__, pkg.DegeneratePair)
        parts.append(ei.value.partial_record)
    assert len(parts[0].objectives) == len(parts[1].objectives) > 0
    assert np.array_equal(parts[0].objectives, parts[1].objectives)
    assert np.array_equal(parts[0].final_iterate, parts[1].final_iterate)
