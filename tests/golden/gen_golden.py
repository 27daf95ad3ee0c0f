"""Generate golden vectors by importing the REAL reference (sobench).

Runs only in the build container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/gen_golden.py

Writes tests/golden/*.npz.  These fixtures pin the oracle (oracle/oracle.py)
and, through it, the CUDA product.  Nothing at test/bench time reads
/root/reference.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import sobench  # noqa: E402
from sobench import _kernels  # noqa: E402
from sobench.backend import make_backend  # noqa: E402
from sobench.bench import gen_meanvar_instance, gen_newsvendor_instance  # noqa: E402
from sobench.frank_wolfe import FwConfig, fw_run  # noqa: E402
from sobench.sampling import (GaussianSpec, RngStream, sample_demands, sample_indices,  # noqa: E402
                              sample_returns, standard_normal, synth_classification, uniform01)
from sobench.sqn import CorrectionPair, SqnConfig, hessian_update, sqn_run  # noqa: E402
from sobench.tasks import (LogisticTask, MeanVarProblem, MeanVarTask, NewsvendorProblem,  # noqa: E402
                           build_sample_set, logistic_gradient, logistic_hvp, logistic_loss,
                           mv_gradient, mv_objective, nv_gradient_hat, nv_objective_exact)

OUT = os.path.dirname(os.path.abspath(__file__))
U128 = (1 << 128) - 1


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    print("wrote", name, {k: np.asarray(v).shape for k, v in arrays.items()})


def split_counter(c):
    m = (1 << 64) - 1
    return np.array([c & m, (c >> 64) & m, c >> 128], dtype=np.uint64)


def rng_cases():
    # (seed, stream_id, counter, n): KAT-like zero key, 64-bit carry, near-2^128
    # counters (span truncation + 256-bit carry inside numpy), odd lengths, >1 span.
    cases = [
        (42, 0, 0, 1000), (0, 0, 0, 17), (7, 2, 3, 65536 + 9),
        ((1 << 64) - 1, (1 << 64) - 1, (1 << 64) - 2, 37),
        (123456789, 5, U128 - 3, 41), (99, 1, U128 - 16384 * 2 + 5, 2 * 65536 + 13),
    ]
    uni = {}
    for i, (seed, sid, ctr, n) in enumerate(cases):
        s = RngStream(seed, sid, ctr)
        u = uniform01(s, n)
        uni[f"u{i}"] = u
        uni[f"u{i}_meta"] = np.array([seed, sid], dtype=np.uint64)
        uni[f"u{i}_ctr"] = split_counter(ctr)
        uni[f"u{i}_after"] = split_counter(s.counter)
    norm_cases = [(42, 1, 0, 1001), (5, 1, 0, 999), (7, 3, (1 << 64) - 3, 21),
                  (11, 1, 0, 65536 + 3)]
    for i, (seed, sid, ctr, n) in enumerate(norm_cases):
        s = RngStream(seed, sid, ctr)
        z = standard_normal(s, n)
        uni[f"z{i}"] = z
        uni[f"z{i}_meta"] = np.array([seed, sid], dtype=np.uint64)
        uni[f"z{i}_ctr"] = split_counter(ctr)
        uni[f"z{i}_after"] = split_counter(s.counter)
    # Random123 known answer: philox4x64_10(ctr=0, key=0), via numpy itself.
    g = np.random.Philox(counter=np.array([(1 << 64) - 1, (1 << 64) - 1, (1 << 64) - 1,
                                           (1 << 64) - 1], dtype=np.uint64),
                         key=np.array([0, 0], dtype=np.uint64))
    uni["kat_zero"] = g.random_raw(4).astype(np.uint64)  # counter wraps to 0 first
    save("rng", **uni)


def tree_cases():
    rng = np.random.default_rng(2024)
    out = {}
    for n in (1, 2, 4095, 4096, 4097, 10_000, 3 * 4096 + 1):
        x = rng.standard_normal(n) * rng.uniform(1e-6, 1e6)
        y = rng.standard_normal(n)
        for chunk in (4096, 3, 64):
            b = make_backend("sequential", chunk_size=chunk)
            out[f"dot_{n}_{chunk}"] = np.array([b.dot(x, y), b.vec_sum(x)])
        out[f"x_{n}"] = x
        out[f"y_{n}"] = y
    for (r, c) in ((9, 5000), (37, 11), (5000, 13), (4097, 3)):
        a = rng.standard_normal((r, c))
        xv = rng.standard_normal(c)
        xt = rng.standard_normal(r)
        out[f"A_{r}x{c}"] = a
        out[f"xv_{r}x{c}"] = xv
        out[f"xt_{r}x{c}"] = xt
        for chunk in (4096, 7):
            b = make_backend("sequential", chunk_size=chunk)
            out[f"mv_{r}x{c}_{chunk}"] = b.matvec(a, xv)
            out[f"mvt_{r}x{c}_{chunk}"] = b.matvec_t(a, xt)
    t = np.concatenate([np.linspace(-750, 750, 301), [0.0, -0.0, 1e-300, -1e-300, 36.0, -36.0]])
    seq = make_backend("sequential")
    out["map_t"] = t
    out["sigmoid"] = seq.map_kernel("sigmoid", t)
    out["exp"] = seq.map_kernel("exp", np.clip(t, -700, 700))
    zl = (rng.uniform(size=t.size) > 0.5).astype(float)
    terms = np.empty(t.size)
    _kernels.logistic_loss_block(t, zl, terms, 0, t.size)
    out["loss_z"] = zl
    out["loss_terms"] = terms
    save("tree", **out)


def meanvar_cases():
    out = {}
    task = gen_meanvar_instance(20, RngStream(42, 0))
    mu, sigma = task.spec.mean, task.spec.diag_std
    out["mu"], out["sigma"] = mu, sigma
    s = RngStream(42, 2)
    x = sample_returns(task.spec, 50, s)
    out["X"] = x
    out["after"] = split_counter(s.counter)
    rng = np.random.default_rng(7)
    w = rng.dirichlet(np.ones(20)) * 0.9
    out["w"] = w
    for chunk in (4096, 16):
        b = make_backend("sequential", chunk_size=chunk)
        ss = build_sample_set(x, b)
        out[f"mean_{chunk}"] = ss.mean
        out[f"Xc_{chunk}"] = ss.centered
        out[f"grad_{chunk}"] = mv_gradient(w, ss, b)
        out[f"obj_{chunk}"] = np.array([mv_objective(w, ss, b)])
    # full FW runs
    for tag, d, epochs, m_inner, n, chunk in (("a", 30, 3, 5, 200, 4096),
                                              ("b", 64, 2, 25, 300, 32)):
        t = gen_meanvar_instance(d, RngStream(42, 0))
        b = make_backend("sequential", chunk_size=chunk)
        prob = MeanVarProblem(t, b)
        cfg = FwConfig(epochs=epochs, inner_iters=m_inner, sample_size=n, stream=RngStream(42, 2))
        rec = fw_run(prob, cfg, b)
        out[f"fw{tag}_cfg"] = np.array([d, epochs, m_inner, n, chunk])
        out[f"fw{tag}_obj"] = rec.objectives
        out[f"fw{tag}_w"] = rec.final_iterate
    save("meanvar", **out)


def newsvendor_cases():
    out = {}
    task = gen_newsvendor_instance(25, RngStream(42, 0))
    for k in ("unit_cost", "holding_cost", "selling_value", "demand_mean", "demand_std",
              "budget_costs"):
        out[k] = getattr(task, k)
    out["budget"] = np.array([task.budget])
    s = RngStream(42, 2)
    dem = sample_demands(task.demand_mean, task.demand_std, 301, s)
    out["demands"] = dem
    out["after"] = split_counter(s.counter)
    rng = np.random.default_rng(9)
    xq = task.demand_mean + task.demand_std * rng.standard_normal(25) * 0.7
    xq[0] = dem[0, 17]          # exact ties with a sample
    xq[1] = -5.0                # below every sample
    xq[2] = 1e9                 # above every sample
    out["xq"] = xq
    seq = make_backend("sequential")
    out["grad"] = nv_gradient_hat(xq, dem, task, seq)
    out["obj"] = np.array([nv_objective_exact(xq, task, seq)])
    for tag, d, epochs, m_inner, n, chunk in (("a", 40, 3, 5, 500, 4096),
                                              ("b", 300, 2, 25, 257, 64)):
        t = gen_newsvendor_instance(d, RngStream(42, 0))
        b = make_backend("sequential", chunk_size=chunk)
        prob = NewsvendorProblem(t, b)
        cfg = FwConfig(epochs=epochs, inner_iters=m_inner, sample_size=n, stream=RngStream(42, 2))
        rec = fw_run(prob, cfg, b)
        out[f"fw{tag}_cfg"] = np.array([d, epochs, m_inner, n, chunk])
        out[f"fw{tag}_obj"] = rec.objectives
        out[f"fw{tag}_x"] = rec.final_iterate
    save("newsvendor", **out)


def logistic_cases():
    out = {}
    s = RngStream(42, 0)
    data = synth_classification(12, s)
    out["X"] = data.features
    out["z"] = data.labels
    out["w_true"] = data.true_weights
    out["after"] = split_counter(s.counter)
    rng = np.random.default_rng(11)
    w = rng.standard_normal(12) * 0.3
    v = rng.standard_normal(12)
    idx = sample_indices(data.n_samples, 50, RngStream(42, 2))
    out["w"], out["v"], out["idx"] = w, v, idx
    seq = make_backend("sequential")
    out["loss_full"] = np.array([logistic_loss(w, data, None, seq)])
    out["loss_idx"] = np.array([logistic_loss(w, data, idx, seq)])
    out["grad_full"] = logistic_gradient(w, data, None, seq)
    out["grad_idx"] = logistic_gradient(w, data, idx, seq)
    out["hvp_full"] = logistic_hvp(w, v, data, None, seq)
    out["hvp_idx"] = logistic_hvp(w, v, data, idx, seq)
    # sample_indices edge cases
    out["si_a"] = sample_indices(1000, 400, RngStream(10, 0))
    out["si_b"] = sample_indices(10, 10, RngStream(9, 0))
    # hessian_update from random SPD-ish pairs
    pairs = []
    for _ in range(4):
        sv = rng.standard_normal(12)
        yv = sv * rng.uniform(0.5, 2.0, 12)
        pairs.append(CorrectionPair(s=sv, y=yv, curvature=seq.dot(sv, yv)))
    h = hessian_update(pairs, 4, 25, seq)
    out["hu_s"] = np.stack([p.s for p in pairs])
    out["hu_y"] = np.stack([p.y for p in pairs])
    out["hu_curv"] = np.array([p.curvature for p in pairs])
    out["hu_H"] = h
    # a full SQN run (d=10, N=300)
    data2 = synth_classification(10, RngStream(42, 0))
    cfg = SqnConfig(pair_every=10, memory=25, beta=2.0, grad_batch=50, hess_batch=100,
                    iterations=60, stream=RngStream(42, 2))
    rec = sqn_run(LogisticTask(data2), cfg, seq)
    out["sqn_obj"] = rec.objectives
    out["sqn_w"] = rec.final_iterate
    save("logistic", **out)


def polytope_cases():
    """lmo_general (lmo.py:92-160) vertices and a multi-resource newsvendor FW trace."""
    from sobench.lmo import PolytopeSet, lmo_general
    from sobench.tasks import NewsvendorTask
    out = {}
    rng = np.random.default_rng(31)
    cases = [(1, 5), (2, 3), (3, 7), (4, 40), (8, 200), (64, 1000), (5, 5)]
    for i, (m, n) in enumerate(cases):
        a = rng.uniform(0.1, 2.0, (m, n))
        c = rng.uniform(0.5, 4.0, m)
        g = rng.standard_normal(n)
        if i == 6:  # ties: equal columns and equal gradient entries (Bland tie-breaks)
            a[:, 3] = a[:, 1]
            g[3] = g[1] = -1.0
            g[0] = 0.0
        out[f"lp{i}_A"], out[f"lp{i}_C"], out[f"lp{i}_g"] = a, c, g
        out[f"lp{i}_s"] = lmo_general(g, PolytopeSet(A=a, C=c))
    base = gen_newsvendor_instance(30, RngStream(42, 0))
    a = rng.uniform(0.5, 2.0, (4, 30))
    cap = 0.3 * (a @ base.demand_mean)
    task = NewsvendorTask(unit_cost=base.unit_cost, holding_cost=base.holding_cost,
                          selling_value=base.selling_value, demand_mean=base.demand_mean,
                          demand_std=base.demand_std, polytope=PolytopeSet(A=a, C=cap))
    for k in ("unit_cost", "holding_cost", "selling_value", "demand_mean", "demand_std"):
        out[f"fw_{k}"] = getattr(task, k)
    out["fw_A"], out["fw_C"] = a, cap
    b = make_backend("sequential")
    rec = fw_run(NewsvendorProblem(task, b), FwConfig(epochs=2, inner_iters=5, sample_size=400,
                                                      stream=RngStream(42, 2)), b)
    out["fw_obj"], out["fw_x"] = rec.objectives, rec.final_iterate
    save("polytope", **out)


if __name__ == "__main__":
    _kernels.warmup()
    which = sys.argv[1:] or ["rng", "tree", "meanvar", "newsvendor", "logistic", "polytope"]
    for name in which:
        globals()[f"{name}_cases"]()
