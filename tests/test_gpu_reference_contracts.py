"""The reference's behavioural contracts (sobench tests/test_{lmo,frank_wolfe,sampling,sqn,
tasks}.py) on the cuda path: edge cases, validation errors and RunAborted semantics.
Each test names the reference test it restates."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2404_11631_b200 as p
    return p


@pytest.fixture(scope="module")
def cuda(pkg):
    return pkg.make_backend("cuda")


# --- lmo (test_lmo.py:32-160) ---------------------------------------------------------------
def test_lmo_simplex_slack_cases(pkg):
    from paper_2404_11631_b200.lmo import lmo_simplex_slack
    np.testing.assert_array_equal(lmo_simplex_slack([-1.0, 2.0, 3.0]), [1.0, 0.0, 0.0])
    np.testing.assert_array_equal(lmo_simplex_slack([1.0, 2.0]), [0.0, 0.0])
    np.testing.assert_array_equal(lmo_simplex_slack([-1.0, -3.0]), [0.0, 1.0])
    np.testing.assert_array_equal(lmo_simplex_slack([-2.0, -2.0]), [1.0, 0.0])   # lowest index
    with pytest.raises(pkg.InvalidGradient):
        lmo_simplex_slack([1.0, np.nan])


def test_lmo_single_budget_cases(pkg):
    from paper_2404_11631_b200.lmo import lmo_single_budget
    np.testing.assert_array_equal(lmo_single_budget([1.0, 1.0], [1.0, 1.0], 4.0), [0.0, 0.0])
    np.testing.assert_array_equal(lmo_single_budget([-1.0], [2.0], 10.0), [5.0])
    with pytest.raises(pkg.InvalidConstraint):
        lmo_single_budget([-1.0, 1.0], [1.0, 0.0], 5.0)
    with pytest.raises(pkg.InvalidGradient):
        lmo_single_budget([-1.0, np.nan], [1.0, 1.0], 5.0)
    rng = np.random.default_rng(3)          # test_against_candidate_enumeration
    for _ in range(100):
        n = int(rng.integers(1, 9))
        g, c, cap = rng.standard_normal(n), rng.uniform(0.5, 2.0, n), float(rng.uniform(1, 5))
        s = lmo_single_budget(g, c, cap)
        cands = [np.zeros(n)] + [np.eye(n)[j] * (cap / c[j]) for j in range(n)]
        assert g @ s <= min(g @ v for v in cands) + 1e-12


# --- frank_wolfe (test_frank_wolfe.py:17-170) ------------------------------------------------
def test_fw_step_size_and_update(pkg, cuda):
    from paper_2404_11631_b200.frank_wolfe import FwState, fw_step_size, fw_update
    assert fw_step_size(0, 25, 0) == 1.0
    assert fw_step_size(2, 25, 0) == 2.0 / 52.0
    with pytest.raises(pkg.ConfigurationError):
        fw_step_size(-1, 25, 0)
    with pytest.raises(pkg.ConfigurationError):
        fw_step_size(0, 25, 25)
    new = fw_update(FwState(np.zeros(3), 0, 0, 10), np.array([0.0, 1.0, 0.0]), cuda)
    np.testing.assert_array_equal(new.iterate, [0.0, 1.0, 0.0])
    assert (new.epoch, new.inner) == (0, 1)
    new = fw_update(FwState(np.zeros(2), 0, 2, 10), np.array([1.0, 0.0]), cuda)
    np.testing.assert_array_equal(new.iterate, [0.5, 0.0])
    new = fw_update(FwState(np.zeros(1), 0, 4, 5), np.zeros(1), cuda)
    assert (new.epoch, new.inner, new.global_step) == (1, 0, 5)


class _ExactQuadratic:
    """test_frank_wolfe.py:63-96: exact moments, host arrays through the cuda backend."""
    name = "exact-quadratic"

    def __init__(self, mean, var, backend):
        self.mean, self.var, self.backend = np.asarray(mean, float), np.asarray(var, float), backend

    @property
    def dimension(self):
        return self.mean.size

    def resample(self, stream, n):
        pass

    def objective(self, w):
        return 0.5 * float(w @ (self.var * w)) - self.backend.dot(w, self.mean)

    def gradient(self, w):
        return self.var * w - self.mean

    def lmo(self, g):
        from paper_2404_11631_b200.lmo import lmo_simplex_slack
        return lmo_simplex_slack(g)

    def check_feasible(self, w):
        return bool(np.all(w >= -1e-10) and w.sum() <= 1 + 1e-10)


def test_fw_infeasible_lmo_output_caught(pkg, cuda):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run

    class Evil(_ExactQuadratic):
        def lmo(self, g):
            return np.full(self.dimension, 5.0)

    cfg = FwConfig(epochs=1, inner_iters=3, sample_size=2, stream=pkg.RngStream(0, 1))
    with pytest.raises(pkg.RunAborted) as exc_info:
        fw_run(Evil(np.ones(3), np.ones(3), cuda), cfg, cuda)
    assert exc_info.value.partial_record is not None


def test_fw_linear_schedule_and_validation(pkg, cuda):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    sizes = []

    class Spy(_ExactQuadratic):
        def resample(self, stream, n):
            sizes.append(n)

    fw_run(Spy(np.ones(2), np.ones(2), cuda),
           FwConfig(epochs=3, inner_iters=2, sample_size=10, stream=pkg.RngStream(0, 1),
                    sample_schedule="linear"), cuda)
    assert sizes == [10, 20, 30]
    with pytest.raises(pkg.ConfigurationError):
        FwConfig(epochs=0, inner_iters=5, sample_size=5, stream=pkg.RngStream(0, 1))


def test_newsvendor_nan_gradient_aborts_with_partial_trace(pkg, cuda):
    """A NaN gradient inside the device loop surfaces as RunAborted(InvalidGradient) with
    the trace up to the failing step (frank_wolfe.py:106-120)."""
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    task = gen_newsvendor_instance(64, pkg.RngStream(42, 0))
    task.selling_value[5] = np.nan               # g_5 = (k - v) + ... is NaN at step 1
    with pytest.raises(pkg.RunAborted) as exc_info:
        fw_run(NewsvendorProblem(task, cuda), FwConfig(2, 5, 500, pkg.RngStream(42, 2)), cuda)
    rec = exc_info.value.partial_record
    assert rec is not None and len(rec.objectives) == 0
    assert isinstance(exc_info.value.__cause__, pkg.InvalidGradient)


# --- sampling (test_sampling.py:60-250) ------------------------------------------------------
def test_sample_returns_validation(pkg, cuda):
    spec = pkg.GaussianSpec(mean=np.zeros(2), diag_std=np.ones(2))
    with pytest.raises(pkg.InsufficientSamples):
        pkg.sample_returns(spec, 1, pkg.RngStream(0, 0), cuda)
    with pytest.raises(pkg.ConfigurationError):
        pkg.GaussianSpec(mean=np.zeros(2))
    with pytest.raises(pkg.InvalidConstraint):
        pkg.GaussianSpec(mean=np.zeros(2), diag_std=np.array([1.0, 0.0]))
    with pytest.raises(pkg.InvalidConstraint):
        pkg.GaussianSpec(mean=np.zeros(2), chol_factor=np.array([[1.0, 0.5], [0.0, 1.0]]))
    sigma = np.array([0.5, 2.0, 1.0])
    a = pkg.sample_returns(pkg.GaussianSpec(mean=np.zeros(3), diag_std=sigma), 20, pkg.RngStream(4, 0), cuda)
    b = pkg.sample_returns(pkg.GaussianSpec(mean=np.zeros(3), chol_factor=np.diag(sigma)), 20,
                           pkg.RngStream(4, 0), cuda)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-15)


def test_sample_demands_contracts(pkg):
    from paper_2404_11631_b200.tasks import sample_demands
    d = sample_demands(np.full(7, 30.0), np.full(7, 15.0), 64, pkg.RngStream(5, 0))
    assert np.all(np.diff(d, axis=1) >= 0)
    d = sample_demands(np.array([30.0]), np.array([1e-12]), 5, pkg.RngStream(6, 0))
    assert np.all(np.abs(d - 30.0) < 1e-10)
    d = sample_demands(np.array([30.0]), np.array([15.0]), 100_000, pkg.RngStream(7, 0))
    assert abs(np.mean(d[0] <= 30.0) - 0.5) < 0.006
    with pytest.raises(pkg.InvalidConstraint):
        sample_demands(np.ones(2), np.array([1.0, -1.0]), 5, pkg.RngStream(0, 0))
    with pytest.raises(pkg.EmptyRequest):
        sample_demands(np.ones(2), np.ones(2), 0, pkg.RngStream(0, 0))


@pytest.mark.parametrize("d,S", [(3, 1000), (5, 4097), (2, 3)])
def test_sample_demands_bitwise_vs_oracle(pkg, d, S):
    """The reference-format demand matrix (sorted rows) equals the oracle's bit for bit,
    and the stream advances as standard_normal(d*S) does."""
    from paper_2404_11631_b200.tasks import sample_demands
    rng = np.random.default_rng(d * S)
    mu, sigma = rng.uniform(20, 50, d), rng.uniform(10, 20, d)
    s = pkg.RngStream(11, 3, 77)
    got = sample_demands(mu, sigma, S, s)
    so = orc.Stream(11, 3, 77)
    z = orc.standard_normal(so, d * S).reshape(d, S)
    want = np.sort(mu[:, None] + sigma[:, None] * z, axis=1)
    assert np.array_equal(got, want)
    assert s.counter == so.counter


def test_sample_indices_contracts(pkg):
    from paper_2404_11631_b200.sampling import sample_indices
    assert sorted(sample_indices(10, 10, pkg.RngStream(9, 0)).tolist()) == list(range(10))
    np.testing.assert_array_equal(sample_indices(1, 1, pkg.RngStream(9, 0)), [0])
    assert len(set(sample_indices(1000, 400, pkg.RngStream(10, 0)).tolist())) == 400
    with pytest.raises(pkg.ConfigurationError):
        sample_indices(5, 6, pkg.RngStream(0, 0))
    with pytest.raises(pkg.ConfigurationError):
        sample_indices(5, 0, pkg.RngStream(0, 0))


# --- sqn / tasks (test_sqn.py:55-215, test_tasks.py:100-345) ---------------------------------
def test_hessian_update_contracts(pkg, cuda):
    from paper_2404_11631_b200.sqn import CorrectionPair, hessian_update
    rng = np.random.default_rng(7)
    s, y = rng.standard_normal(12), rng.standard_normal(12)
    y = y + 3.0 * s                                   # positive curvature
    pair = CorrectionPair(s=torch.from_numpy(s).cuda(), y=torch.from_numpy(y).cuda(),
                          curvature=float(s @ y))
    h = hessian_update([pair], t=1, memory=1, backend=cuda).cpu().numpy()
    np.testing.assert_allclose(h @ y, s, atol=1e-10 * (1 + np.abs(s).max()))   # secant
    with pytest.raises(pkg.DegeneratePair):
        hessian_update([CorrectionPair(torch.ones(3, dtype=torch.float64, device="cuda"),
                                       torch.zeros(3, dtype=torch.float64, device="cuda"), 0.0)],
                       t=1, memory=5, backend=cuda)
    with pytest.raises(pkg.ConfigurationError):
        hessian_update([], t=1, memory=5, backend=cuda)
    with pytest.raises(pkg.ConfigurationError):
        hessian_update([pair, pair], t=1, memory=5, backend=cuda)


def test_sqn_config_validation(pkg):
    from paper_2404_11631_b200.sqn import SqnConfig
    with pytest.raises(pkg.ConfigurationError):
        SqnConfig(pair_every=0, memory=1, beta=1.0, grad_batch=1, hess_batch=1, iterations=1,
                  stream=pkg.RngStream(0, 0))
    with pytest.raises(pkg.ConfigurationError):
        SqnConfig(pair_every=1, memory=1, beta=0.0, grad_batch=1, hess_batch=1, iterations=1,
                  stream=pkg.RngStream(0, 0))


def test_task_validation_errors(pkg, cuda):
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200 import tasks as T
    with pytest.raises(pkg.InsufficientSamples):
        T.build_sample_set(np.ones((1, 3)), cuda)
    task = gen_newsvendor_instance(2, pkg.RngStream(1, 0))
    with pytest.raises(pkg.InsufficientSamples):
        T.nv_gradient_hat(np.zeros(2), np.empty((2, 0)), task, cuda)
    data = synth_classification(4, pkg.RngStream(15, 0))
    with pytest.raises(pkg.DimensionMismatch):
        T.logistic_loss(np.zeros(5), data, None, cuda)
