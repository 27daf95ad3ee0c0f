"""GPU parity for the newsvendor hot path: resample layout, ECDF counts, FW traces."""
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


def _task_from_golden(pkg, g):
    from paper_2404_11631_b200.tasks import NewsvendorTask
    return NewsvendorTask(unit_cost=g["unit_cost"], holding_cost=g["holding_cost"],
                          selling_value=g["selling_value"], demand_mean=g["demand_mean"],
                          demand_std=g["demand_std"], budget_costs=g["budget_costs"],
                          budget=float(g["budget"][0]))


def _check_layout(dev, sorted_rows):
    """Keyed segments decode to exactly the reference's sorted rows; bucket order respected."""
    from paper_2404_11631_b200.tasks import nv_geometry
    seg, nb = nv_geometry()
    d, S = sorted_rows.shape
    dem = dev.decode().cpu().numpy()
    assert np.array_equal(np.sort(dem, axis=1), sorted_rows)
    keys = dev.keys.view(d, S).cpu().numpy().view(np.uint32).astype(np.int64)
    off = dev.off.view(d, dev.nseg, nb).cpu().numpy().astype(np.int64) & 0xFFFF
    for j in range(min(d, 64)):
        for s in range(dev.nseg):
            kv = keys[j, s * seg:(s + 1) * seg]
            b = kv >> 22
            assert np.all(np.diff(b) >= 0)
            assert np.array_equal(np.sort(kv & 4095), np.arange(kv.size))  # each draw once
            assert np.array_equal(off[j, s], np.searchsorted(b, np.arange(nb), side="left"))


def test_resample_matches_reference_rows(pkg, golden):
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    g = golden("newsvendor")
    prob = NewsvendorProblem(_task_from_golden(pkg, g), pkg.make_backend("cuda"))
    s = pkg.RngStream(42, 2)
    prob.resample(s, 301)
    assert s.counter == counter_of(g["after"])
    _check_layout(prob.dev, g["demands"])
    # ECDF gradient at the golden query points (ties, below-all, above-all included)
    got = prob.gradient(g["xq"])
    assert np.array_equal(got, g["grad"])


# counters: word-0 fast path (77; high word set), and a draw carrying into word 1
@pytest.mark.parametrize("d,S,ctr", [(300, 5000, 77), (64, 100_000, 77), (1000, 4096, 77),
                                     (7, 12289, 77), (5, 3, 77), (300, 5000, (5 << 64) + 3),
                                     (300, 5000, (1 << 64) - 100)])
def test_counts_vs_oracle(pkg, d, S, ctr):
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    task = gen_newsvendor_instance(d, pkg.RngStream(42, 0))
    prob = NewsvendorProblem(task, pkg.make_backend("cuda"))
    prob.resample(pkg.RngStream(42, 2, ctr), S)
    want_rows = orc.sample_demands(task.demand_mean, task.demand_std, S, orc.Stream(42, 2, ctr))
    _check_layout(prob.dev, want_rows)
    rng = np.random.default_rng(d)
    for trial in range(4):
        x = task.demand_mean + task.demand_std * rng.standard_normal(d) * (0.5 + trial)
        if trial == 0:  # exact ties with samples
            x = want_rows[np.arange(d), rng.integers(0, S, d)]
        if trial == 1:
            x[: d // 2] = 0.0
        cnt = prob.dev.counts(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(cnt, orc.ecdf_counts(want_rows, x))


@pytest.mark.parametrize("tag", ["a", "b"])
def test_fw_trace_golden(pkg, golden, tag):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    g = golden("newsvendor")
    d, epochs, m_inner, n, chunk = (int(v) for v in g[f"fw{tag}_cfg"])
    b = pkg.make_backend("cuda", chunk_size=chunk)
    task = gen_newsvendor_instance(d, pkg.RngStream(42, 0))
    rec = fw_run(NewsvendorProblem(task, b), FwConfig(epochs, m_inner, n, pkg.RngStream(42, 2)), b)
    assert np.array_equal(rec.final_iterate, g[f"fw{tag}_x"])
    assert np.array_equal(rec.iterations, np.arange(1, epochs * m_inner + 1))
    assert np.array_equal(rec.objectives, g[f"fw{tag}_obj"])  # glibc-exact erf/exp terms
    assert np.all(np.diff(rec.elapsed_ns) >= 0)


def test_fw_trace_vs_oracle_large(pkg):
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    d, S, K, M = 2000, 20_000, 2, 25
    b = pkg.make_backend("cuda")
    task = gen_newsvendor_instance(d, pkg.RngStream(42, 0))
    rec = fw_run(NewsvendorProblem(task, b), FwConfig(K, M, S, pkg.RngStream(42, 2)), b)
    ot = orc.gen_newsvendor_instance(d, orc.Stream(42, 0))
    objs, x = orc.fw_run_newsvendor(ot, K, M, S, orc.Stream(42, 2))
    assert np.array_equal(rec.final_iterate, x)
    assert np.array_equal(rec.objectives, objs)


def test_reference_fw_loop_drives_device_problem(pkg, golden):
    """The duck-typed protocol (host arrays) gives the same trace as the fused path."""
    from paper_2404_11631_b200.frank_wolfe import FwConfig
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    from paper_2404_11631_b200 import frank_wolfe as fwm
    g = golden("newsvendor")
    d, epochs, m_inner, n, chunk = (int(v) for v in g["fwa_cfg"])
    b = pkg.make_backend("cuda", chunk_size=chunk)
    prob = NewsvendorProblem(gen_newsvendor_instance(d, pkg.RngStream(42, 0)), b)

    class HostOnly:  # hide fw_run_device -> generic reference loop
        name = "newsvendor"
        dimension = prob.dimension
        resample = prob.resample
        gradient = prob.gradient
        lmo = prob.lmo
        check_feasible = prob.check_feasible
        objective = prob.objective

    rec = fwm.fw_run(HostOnly(), FwConfig(epochs, m_inner, n, pkg.RngStream(42, 2)), b)
    assert np.array_equal(rec.final_iterate, g["fwa_x"])
    assert np.array_equal(rec.objectives, g["fwa_obj"])


def test_degenerate_sigma_counts(pkg):
    """sigma = 1e-12 (tests/test_sampling.py:156-158): every draw is ambiguous -> exact path."""
    from paper_2404_11631_b200.tasks import NewsvendorProblem, NewsvendorTask
    task = NewsvendorTask(unit_cost=[1.0, 1.5], holding_cost=[0.5, 0.5], selling_value=[3.0, 4.0],
                          demand_mean=[30.0, 25.0], demand_std=[1e-12, 3.0], budget_costs=[1.0, 1.0],
                          budget=20.0)
    prob = NewsvendorProblem(task, pkg.make_backend("cuda"))
    prob.resample(pkg.RngStream(6, 0), 997)
    rows = orc.sample_demands(task.demand_mean, task.demand_std, 997, orc.Stream(6, 0))
    for x0 in (30.0, 30.0 + 1e-13, 25.0, np.nextafter(30.0, 0.0)):
        x = np.array([x0, x0])
        cnt = prob.dev.counts(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(cnt, orc.ecdf_counts(rows, x))


def test_approximation_error_bound(pkg):
    """The fp32 approximation error stays far inside NV_EPSZ = 1e-4 over 2^26 draws."""
    from paper_2404_11631_b200.tasks import NewsvendorProblem, NewsvendorTask
    d, S = 64, 1 << 20
    ones = np.ones(d)
    task = NewsvendorTask(unit_cost=ones, holding_cost=ones, selling_value=3 * ones,
                          demand_mean=np.zeros(d), demand_std=ones, budget_costs=ones, budget=1.0)
    prob = NewsvendorProblem(task, pkg.make_backend("cuda"))
    prob.resample(pkg.RngStream(123, 9), S)
    exact = prob.dev.decode()                       # D = 0 + 1*z, storage order
    keys = prob.dev.keys.view(d, S).long() & 0xFFFFFFFF
    q = (keys >> 12).double()
    lo = (q - 1.0) * (19.0 / 2 ** 20) - 9.5
    hi = (q + 2.0) * (19.0 / 2 ** 20) - 9.5
    inside = (exact >= lo - 1e-5) & (exact <= hi + 1e-5)
    assert bool(inside.all())


@pytest.mark.parametrize("seed,sid,ctr", [(42, 2, 0), (7, 1, (1 << 64) - 3)])
def test_approximation_error_measured(pkg, seed, sid, ctr):
    """max |z~ - z| over 2^28 normals stays below a third of the bound the queries assume."""
    import ctypes
    from paper_2404_11631_b200 import _lib
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    eps = ctypes.c_double()
    s = pkg.RngStream(seed, sid, ctr)
    _lib.call("simopt_nv_approx_error", _lib.stream_ptr(), *s.words(), 1 << 28, _lib.ptr(out),
              ctypes.byref(eps))
    m = float(out.item())
    print(f"max |z~ - z| = {m:.3e} (bound {eps.value:.1e})")
    assert m < eps.value / 3


def test_graph_engine_matches_eager(pkg):
    """Epochs replayed as CUDA graphs (parity graphs, device-resident gamma/draw) give the
    eager engine's trace bit for bit."""
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.records import TraceBuilder
    from paper_2404_11631_b200.tasks import NewsvendorProblem, make_nv_engine
    task = gen_newsvendor_instance(700, pkg.RngStream(42, 0))
    out = []
    for graph in (False, True):
        prob = NewsvendorProblem(task, pkg.make_backend("cuda"))
        K, M, S = 5, 6, 3000
        eng = make_nv_engine(prob, M, K, 4096, graph=graph)
        stream = pkg.RngStream(42, 2)
        eng.start()
        for k in range(K):
            eng.enqueue_epoch(k, stream, S, next_samples=S if k + 1 < K else None)
        eng.finish()
        tr = TraceBuilder()
        for k in range(K):
            assert eng.check_epoch(k, tr) is None
        out.append((tr.build("nv", 700, "cuda", 0, 42, None).objectives, eng.iterate(K * M).cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_graph_engine_linear_schedule(pkg):
    """A linear sample schedule changes S (and reallocates the layout slots) every epoch:
    the graph engine re-captures per layout and still gives the oracle's trace bit for bit."""
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.records import TraceBuilder
    from paper_2404_11631_b200.tasks import NewsvendorProblem, make_nv_engine
    d, K, M, S = 333, 5, 4, 1500
    task = gen_newsvendor_instance(d, pkg.RngStream(42, 0))
    for graph in (False, True):
        prob = NewsvendorProblem(task, pkg.make_backend("cuda"))
        eng = make_nv_engine(prob, M, K, 4096, graph=graph)
        stream = pkg.RngStream(42, 2)
        eng.start()
        for k in range(K):
            eng.enqueue_epoch(k, stream, S * (k + 1), next_samples=S * (k + 2) if k + 1 < K else None)
        eng.finish()
        tr = TraceBuilder()
        for k in range(K):
            assert eng.check_epoch(k, tr) is None
        objs, x = orc.fw_run_newsvendor(orc.gen_newsvendor_instance(d, orc.Stream(42, 0)), K, M, S,
                                        orc.Stream(42, 2), schedule="linear")
        assert np.array_equal(eng.iterate(K * M).cpu().numpy(), x), graph
        np.testing.assert_allclose(tr.build("nv", d, "cuda", 0, 42, None).objectives, objs, rtol=1e-13)


def test_graph_engine_epoch_start_iterate(pkg):
    """RunAborted's final_iterate for a failure at an epoch's first step is the epoch's
    starting iterate, even while the next epoch (whose ring parity holds it) runs: the
    check of epoch k-1 happens after epoch k is enqueued, as in _nv_fw_run_device."""
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem, make_nv_engine
    d, K, M, S = 300, 4, 3, 2000
    task = gen_newsvendor_instance(d, pkg.RngStream(42, 0))
    otask = orc.gen_newsvendor_instance(d, orc.Stream(42, 0))
    want = [np.zeros(d)] + [orc.fw_run_newsvendor(otask, k, M, S, orc.Stream(42, 2))[1]
                            for k in range(1, K + 1)]
    eng = make_nv_engine(NewsvendorProblem(task, pkg.make_backend("cuda")), M, K, 4096, graph=True)
    stream = pkg.RngStream(42, 2)
    eng.start()
    for k in range(K):
        eng.enqueue_epoch(k, stream, S, next_samples=S if k + 1 < K else None)
        if k >= 1:
            torch.cuda.synchronize()
            assert np.array_equal(eng.iterate((k - 1) * M, k - 1).cpu().numpy(), want[k - 1]), k
            assert np.array_equal(eng.iterate(k * M, k - 1).cpu().numpy(), want[k]), k
    eng.finish()


@pytest.mark.parametrize("d,S", [(2000, 100_000), (301, 5001), (64, 4096), (7, 3)])
def test_resample_kernels_agree(pkg, d, S, monkeypatch):
    """The warp-specialised resample (default) and the single-role kernel write the same
    layout: identical bucket starts, and the same keys inside every bucket."""
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    prob = NewsvendorProblem(gen_newsvendor_instance(d, pkg.RngStream(42, 0)), pkg.make_backend("cuda"))
    out = []
    for variant in ("1", "0"):
        monkeypatch.setenv("SIMOPT_NV_RESAMPLE", variant)
        prob.dev.resample(pkg.RngStream(9, 4, (1 << 64) - 1000), S)   # 64-bit carry path too
        keys = (prob.dev.keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).view(d, S)
        canon = torch.cat([torch.sort(keys[:, s0:s0 + 4096], dim=1).values for s0 in range(0, S, 4096)], 1)
        out.append((prob.dev.off.clone(), canon))
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])


@pytest.mark.parametrize("d,chunk,H,r0,M", [(10_000, 4096, 51, 40, 25), (3_001, 16, 7, 5, 6),
                                            (1, 4096, 3, 2, 3), (5_000, 7, 4, 0, 4)])
def test_epoch_records_match_per_step_sums(pkg, d, chunk, H, r0, M):
    """simopt_nv_epoch_records = per step nv_cost_terms + tree_sums2, bit for bit (ring
    wrap, chunk counts 1..715 incl. > 64, a ragged last chunk, one product)."""
    from paper_2404_11631_b200 import _lib
    g = torch.Generator().manual_seed(d + chunk)
    xs = (torch.rand(H, d, generator=g, dtype=torch.float64) * 50).cuda()
    mu = (torch.rand(d, generator=g, dtype=torch.float64) * 40 + 5).cuda()
    sd = (torch.rand(d, generator=g, dtype=torch.float64) * 10 + 0.5).cuda()
    c, k, h, v = ((torch.rand(d, generator=g, dtype=torch.float64) * 3).cuda() for _ in range(4))
    spent, objs = torch.empty(M, dtype=torch.float64, device="cuda"), torch.empty(M, dtype=torch.float64, device="cuda")
    P = _lib.ptr
    _lib.call("simopt_nv_epoch_records", _lib.stream_ptr(), P(xs), H, r0, M, P(c), P(mu), P(sd),
              P(k), P(h), P(v), d, chunk, P(spent), P(objs))
    terms = torch.empty(d, dtype=torch.float64, device="cuda")
    ref = torch.empty(2, M, dtype=torch.float64, device="cuda")
    for m in range(M):
        x = xs[(r0 + m) % H]
        _lib.call("simopt_nv_cost_terms", _lib.stream_ptr(), P(x), P(mu), P(sd), P(k), P(h), P(v), d, P(terms))
        _lib.call("simopt_tree_sums2", _lib.stream_ptr(), P(c), P(x), d, P(ref[0, m:]), P(terms), None, d,
                  P(ref[1, m:]), chunk)
    assert torch.equal(spent, ref[0]) and torch.equal(objs, ref[1])


@pytest.mark.parametrize("qcap", ["0", "1"])
def test_step_queue_overflow_path(qcap):
    """Ambiguous draws that do not fit the step kernel's CTA queue are resolved by the warp
    that found them: with the queue shrunk to 0/1 entries (SIMOPT_NV_QCAP) FW traces still
    match the oracle bit for bit (scalar and 16-byte key-load paths)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SIMOPT_NV_QCAP=qcap)
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_paths.py"), "nv"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "nv ok" in r.stdout, r.stdout + r.stderr
