"""Multi-resource newsvendor: the device simplex LMO (csrc/lp.cu) against the reference's
lmo_general vertices (tests/golden/polytope.npz, made by importing sobench) and the oracle
restatement; the FW trace of a polytope newsvendor run bit for bit."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2404_11631_b200 as p
    return p


@pytest.mark.parametrize("i", range(7))
def test_lmo_general_golden(pkg, golden, i):
    from paper_2404_11631_b200.lmo import PolytopeSet, lmo_general
    g = golden("polytope")
    s = lmo_general(g[f"lp{i}_g"], PolytopeSet(A=g[f"lp{i}_A"], C=g[f"lp{i}_C"]))
    assert np.array_equal(s, g[f"lp{i}_s"])


@pytest.mark.parametrize("m,n,seed", [(1, 1, 0), (2, 3, 1), (16, 500, 2), (64, 10_000, 3),
                                      (7, 7, 4)])
def test_lmo_general_vs_oracle(pkg, m, n, seed):
    from paper_2404_11631_b200.lmo import PolytopeSet, lmo_general
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.05, 3.0, (m, n))
    c = rng.uniform(0.2, 5.0, m)
    for _ in range(3):
        g = rng.standard_normal(n)
        g[rng.integers(0, n)] = 0.0
        s = lmo_general(g, PolytopeSet(A=a, C=c))
        assert np.array_equal(s, orc.lmo_general(g, a, c))
        assert np.all(s >= -1e-10) and np.all(a @ s <= c * (1 + 1e-10) + 1e-10)


def test_lmo_general_errors(pkg):
    from paper_2404_11631_b200.lmo import PolytopeSet, lmo_general
    pset = PolytopeSet(A=np.ones((1, 3)), C=np.ones(1))
    with pytest.raises(pkg.DimensionMismatch):
        lmo_general(np.ones(4), pset)
    with pytest.raises(pkg.SolverStall):
        lmo_general(np.array([-1.0, -2.0, -3.0]), pset, max_iters=0)
    with pytest.raises(pkg.InvalidGradient):
        lmo_general(np.array([-1.0, np.nan, 0.0]), pset)
    np.testing.assert_array_equal(
        lmo_general([0.5, 1.0], PolytopeSet(A=np.array([[1.0, 2.0], [2.0, 1.0]]), C=np.array([3.0, 3.0]))),
        [0.0, 0.0])
    with pytest.raises(pkg.InvalidConstraint):
        PolytopeSet(A=np.array([[1.0, -0.1]]), C=np.array([1.0]))
    with pytest.raises(pkg.InvalidConstraint):
        PolytopeSet(A=np.array([[1.0, 1.0]]), C=np.array([0.0]))


def test_newsvendor_polytope_fw_trace_golden(pkg, golden):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.lmo import PolytopeSet
    from paper_2404_11631_b200.tasks import NewsvendorProblem, NewsvendorTask
    g = golden("polytope")
    task = NewsvendorTask(unit_cost=g["fw_unit_cost"], holding_cost=g["fw_holding_cost"],
                          selling_value=g["fw_selling_value"], demand_mean=g["fw_demand_mean"],
                          demand_std=g["fw_demand_std"], polytope=PolytopeSet(A=g["fw_A"], C=g["fw_C"]))
    b = pkg.make_backend("cuda")
    rec = fw_run(NewsvendorProblem(task, b), FwConfig(2, 5, 400, pkg.RngStream(42, 2)), b)
    assert np.array_equal(rec.final_iterate, g["fw_x"])                 # iterates bit-exact
    assert np.array_equal(rec.objectives, g["fw_obj"])
