"""CPU oracle for the sobench hot path -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference algorithms (arXiv 2404.11631 artifact
``sobench``; paths below are relative to /root/reference/pkg/src/sobench)
on top of the C kernels in ``oracle.c``.  Composition follows the reference
line by line (same numpy elementwise expressions, same association), so that
the results are bit-identical to the reference.  That claim is pinned by
``tests/test_oracle.py`` against golden vectors that ``tests/golden/gen_golden.py``
produced by importing the reference itself.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference legs may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

CHUNK = 4096            # backend.py:27
FEAS_TOL = 1e-10        # tasks.py:27
CURVATURE_RTOL = 1e-10  # sqn.py:34
_U64 = (1 << 64) - 1

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        u64, i64, d = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
        L.orc_uniform01.argtypes = [u64, u64, u64, u64, i64, _dp]
        L.orc_standard_normal.argtypes = [u64, u64, u64, u64, i64, _dp]
        L.orc_philox_block.argtypes = [_u64p, _u64p, _u64p]
        L.orc_boxmuller.argtypes = [_dp, _dp, i64]
        L.orc_dot.argtypes = [_dp, _dp, i64, i64]
        L.orc_dot.restype = d
        L.orc_vec_sum.argtypes = [_dp, i64, i64]
        L.orc_vec_sum.restype = d
        L.orc_fold_pairwise.argtypes = [_dp, i64]
        L.orc_fold_pairwise.restype = d
        L.orc_matvec.argtypes = [_dp, i64, i64, _dp, _dp, i64]
        L.orc_matvec_t.argtypes = [_dp, i64, i64, _dp, _dp, i64]
        L.orc_sigmoid.argtypes = [_dp, _dp, i64]
        L.orc_exp.argtypes = [_dp, _dp, i64]
        L.orc_logistic_loss_terms.argtypes = [_dp, _dp, _dp, i64]
        L.orc_normal_cdf.argtypes = [_dp, _dp, i64]
        L.orc_newsvendor_cost.argtypes = [_dp] * 7 + [i64]
        L.orc_ecdf_count.argtypes = [_dp, i64, i64, _dp, _i64p]
        L.orc_bfgs_rank2.argtypes = [_dp, _dp, _dp, d, d, i64]
        L.orc_sort_rows.argtypes = [_dp, i64, i64]
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.orc_philox4x32.argtypes = [u32p, u32p, i64, u32p]
        L.orc_sfc64.argtypes = [_u64p, i64, _u64p]
        L.orc_xoshiro256pp.argtypes = [_u64p, i64, _u64p]
        L.orc_xoshiro256pp_jump.argtypes = [_u64p]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp)


def _vec(x):
    return np.ascontiguousarray(x, dtype=np.float64)


# ---------------------------------------------------------------- RNG
@dataclass
class Stream:
    """RngStream (sampling.py:51-80): (seed, stream_id, 128-bit block counter)."""
    seed: int
    stream_id: int
    counter: int = 0

    def clone(self):
        return Stream(self.seed, self.stream_id, self.counter)


def uniform01(stream: Stream, n: int) -> np.ndarray:
    """sampling.py:87-102."""
    out = np.empty(n)
    c = stream.counter
    lib().orc_uniform01(stream.seed, stream.stream_id, c & _U64, (c >> 64) & _U64, n, _p(out))
    stream.counter += (n + 3) // 4
    return out


def standard_normal(stream: Stream, n: int) -> np.ndarray:
    """sampling.py:105-120 (Box-Muller on 2*ceil(n/2) uniforms)."""
    out = np.empty(n)
    c = stream.counter
    lib().orc_standard_normal(stream.seed, stream.stream_id, c & _U64, (c >> 64) & _U64, n,
                              _p(out))
    m = 2 * ((n + 1) // 2)
    stream.counter += (m + 3) // 4
    return out


def philox_block(ctr4, key2):
    c = (ctypes.c_uint64 * 4)(*ctr4)
    k = (ctypes.c_uint64 * 2)(*key2)
    o = (ctypes.c_uint64 * 4)()
    lib().orc_philox_block(c, k, o)
    return list(o)


# ---------------------------------------------------------------- backend
def dot(x, y, chunk=CHUNK) -> float:
    x, y = _vec(x), _vec(y)
    return float(lib().orc_dot(_p(x), _p(y), x.size, chunk))


def vec_sum(x, chunk=CHUNK) -> float:
    x = _vec(x)
    return float(lib().orc_vec_sum(_p(x), x.size, chunk))


def matvec(a, x, chunk=CHUNK) -> np.ndarray:
    a, x = np.ascontiguousarray(a, dtype=np.float64), _vec(x)
    out = np.empty(a.shape[0])
    lib().orc_matvec(_p(a), a.shape[0], a.shape[1], _p(x), _p(out), chunk)
    return out


def matvec_t(a, x, chunk=CHUNK) -> np.ndarray:
    a, x = np.ascontiguousarray(a, dtype=np.float64), _vec(x)
    out = np.empty(a.shape[1])
    lib().orc_matvec_t(_p(a), a.shape[0], a.shape[1], _p(x), _p(out), chunk)
    return out


def axpy(alpha, x, y):
    return alpha * _vec(x) + _vec(y)  # backend.py:127-132


def sigmoid(x):
    x = _vec(x)
    out = np.empty(x.size)
    lib().orc_sigmoid(_p(x), _p(out), x.size)
    return out


def exp(x):
    x = _vec(x)
    out = np.empty(x.size)
    lib().orc_exp(_p(x), _p(out), x.size)
    return out


def map_kernel(kernel, x):
    if kernel == "negate":
        return np.negative(_vec(x))
    return {"sigmoid": sigmoid, "exp": exp}[kernel](x)


# ---------------------------------------------------------------- task 1: meanvar
def sample_returns_diag(mu, sigma, n_samples, stream):
    """sampling.py:156-166 (diag path)."""
    d = mu.size
    z = standard_normal(stream, n_samples * d).reshape(n_samples, d)
    return mu[None, :] + sigma[None, :] * z


def build_sample_set(samples, chunk=CHUNK):
    """tasks.py:56-64 -> (mean, centered)."""
    n = samples.shape[0]
    col_sums = matvec_t(samples, np.ones(n), chunk)
    mean = col_sums * (1.0 / n)
    return mean, samples - mean[None, :]


def mv_objective(w, mean, centered, chunk=CHUNK):
    """tasks.py:67-75."""
    q = matvec(centered, w, chunk)
    quad = dot(q, q, chunk)
    lin = dot(w, mean, chunk)
    return 0.5 * quad / (centered.shape[0] - 1) - lin


def mv_gradient(w, mean, centered, chunk=CHUNK):
    """tasks.py:78-85."""
    q = matvec(centered, w, chunk)
    gq = matvec_t(centered, q, chunk)
    return gq * (1.0 / (centered.shape[0] - 1)) - mean


# ---------------------------------------------------------------- task 2: newsvendor
def sample_demands(mu, sigma, n_samples, stream):
    """sampling.py:173-193 (rows sorted ascending)."""
    z = standard_normal(stream, mu.size * n_samples).reshape(mu.size, n_samples)
    d = mu[:, None] + sigma[:, None] * z
    d.sort(axis=1)
    return d


def ecdf_counts(demands, x):
    x = _vec(x)
    out = np.empty(x.size, np.int64)
    lib().orc_ecdf_count(_p(demands), demands.shape[0], demands.shape[1], _p(x),
                         out.ctypes.data_as(_i64p))
    return out


def nv_gradient_hat(x, demands, k, h, v):
    """tasks.py:141-160."""
    counts = ecdf_counts(demands, x)
    frac = counts / demands.shape[1]
    return k - v + (h + v) * frac


def nv_cost_terms(x, mu, sigma, k, h, v):
    x = _vec(x)
    out = np.empty(x.size)
    lib().orc_newsvendor_cost(_p(x), _p(mu), _p(sigma), _p(k), _p(h), _p(v), _p(out), x.size)
    return out


def nv_objective_exact(x, mu, sigma, k, h, v, chunk=CHUNK):
    """tasks.py:174-188."""
    return vec_sum(nv_cost_terms(x, mu, sigma, k, h, v), chunk)


def normal_cdf(z):
    z = _vec(z)
    out = np.empty(z.size)
    lib().orc_normal_cdf(_p(z), _p(out), z.size)
    return out


def nv_gradient_exact(x, mu, sigma, k, h, v):
    """tasks.py:163-171."""
    z = (_vec(x) - mu) / sigma
    return k - v + (h + v) * normal_cdf(z)


# ---------------------------------------------------------------- LMOs / FW
class InvalidGradientError(ValueError):
    pass


def lmo_simplex_slack(g):
    """lmo.py:56-65."""
    g = _vec(g)
    if np.isnan(g).any():
        raise InvalidGradientError("gradient contains NaN")
    s = np.zeros(g.size)
    j = int(np.argmin(g))
    if g[j] < 0.0:
        s[j] = 1.0
    return s


def lmo_single_budget(g, c, budget):
    """lmo.py:68-89."""
    g = _vec(g)
    if np.isnan(g).any():
        raise InvalidGradientError("gradient contains NaN")
    vals = g * (budget / c)
    j = int(np.argmin(vals))
    s = np.zeros(g.size)
    if g[j] < 0.0:
        s[j] = budget / c[j]
    return s


def fw_step_size(epoch, inner_iters, inner):
    return 2.0 / (epoch * inner_iters + inner + 2)  # frank_wolfe.py:62-66


def fw_update(w, s, epoch, inner_iters, inner):
    """frank_wolfe.py:69-82 -> new iterate."""
    gamma = fw_step_size(epoch, inner_iters, inner)
    direction = axpy(-1.0, w, s)
    return axpy(gamma, direction, w)


def fw_run_meanvar(mu, sigma, epochs, inner_iters, n_samples, stream, chunk=CHUNK):
    """frank_wolfe.py:91-121 driving MeanVarProblem (tasks.py:261-290)."""
    d = mu.size
    w = np.zeros(d)
    objs = []
    for k in range(epochs):
        x = sample_returns_diag(mu, sigma, n_samples, stream)
        mean, xc = build_sample_set(x, chunk)
        for m in range(inner_iters):
            g = mv_gradient(w, mean, xc, chunk)
            s = lmo_simplex_slack(g)
            w = fw_update(w, s, k, inner_iters, m)
            if not (np.all(w >= -FEAS_TOL) and np.sum(w) <= 1.0 + FEAS_TOL):
                raise RuntimeError("infeasible")
            objs.append(mv_objective(w, mean, xc, chunk))
    return np.array(objs), w


def fw_run_newsvendor(task, epochs, inner_iters, n_samples, stream, chunk=CHUNK,
                      schedule="constant"):
    """frank_wolfe.py:91-121 driving NewsvendorProblem (tasks.py:293-334); `schedule`
    is FwConfig.sample_schedule (frank_wolfe.py:41-46: "linear" draws n*(k+1) in epoch k)."""
    mu, sigma, k_, h, v, c, budget = (task[n] for n in ("mu", "sigma", "k", "h", "v", "c",
                                                        "budget"))
    d = mu.size
    x = np.zeros(d)
    objs = []
    for k in range(epochs):
        n_k = n_samples * (k + 1) if schedule == "linear" else n_samples
        dem = sample_demands(mu, sigma, n_k, stream)
        for m in range(inner_iters):
            g = nv_gradient_hat(x, dem, k_, h, v)
            s = lmo_single_budget(g, c, budget)
            x = fw_update(x, s, k, inner_iters, m)
            if np.any(x < -FEAS_TOL) or dot(c, x, chunk) > budget * (1.0 + FEAS_TOL):
                raise RuntimeError("infeasible")
            objs.append(nv_objective_exact(x, mu, sigma, k_, h, v, chunk))
    return np.array(objs), x


def lmo_general(g, a, c, max_iters=None):
    """lmo.py:92-160: dense primal simplex over {a s <= c, s >= 0} from the slack basis,
    Bland's rule.  Row operations are whole-row numpy expressions with the reference's
    association (row /= piv; row_i -= f_i * row_leave; cost -= c_e * row_leave).
    Returns s, or raises ValueError("nan" | "unbounded" | "cap")."""
    g = np.ascontiguousarray(g, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    m, n = a.shape
    if np.isnan(g).any():
        raise ValueError("nan")
    cap = 10 * (n + m) if max_iters is None else max_iters
    width = n + m
    t = np.concatenate([a, np.eye(m), c[:, None]], axis=1)
    red = np.concatenate([g, np.zeros(m)])
    basic = np.arange(n, n + m)
    tol_in = 1e-12 * (1.0 + float(np.max(np.abs(g))))
    for _ in range(cap):
        below = np.nonzero(red < -tol_in)[0]
        if below.size == 0:
            break
        e = int(below[0])
        leave, best = -1, np.inf
        for i in range(m):
            col = t[i, e]
            if col > 1e-12:
                r = t[i, -1] / col
                tie = abs(r - best) <= 1e-15 and (leave < 0 or basic[i] < basic[leave])
                if r < best - 1e-15 or tie:
                    best, leave = r, i
        if leave < 0:
            raise ValueError("unbounded")
        t[leave] = t[leave] / t[leave, e]
        prow = t[leave]
        for i in range(m):
            f = t[i, e]
            if i != leave and f != 0.0:
                t[i] = t[i] - f * prow
        ce = red[e]
        if ce != 0.0:
            red = red - ce * prow[:width]
        basic[leave] = e
    else:
        raise ValueError("cap")
    s = np.zeros(n)
    for i, b in enumerate(basic):
        if b < n:
            s[b] = t[i, -1]
    return s


def fw_run_newsvendor_polytope(task, a, c, epochs, inner_iters, n_samples, stream, chunk=CHUNK):
    """fw_run over NewsvendorProblem with a polytope (tasks.py:321-334)."""
    mu, sigma, k_, h, v = (task[n] for n in ("mu", "sigma", "k", "h", "v"))
    x = np.zeros(mu.size)
    objs = []
    for k in range(epochs):
        dem = sample_demands(mu, sigma, n_samples, stream)
        for m in range(inner_iters):
            g = nv_gradient_hat(x, dem, k_, h, v)
            s = lmo_general(g, a, c)
            x = fw_update(x, s, k, inner_iters, m)
            if np.any(x < -FEAS_TOL) or np.any(matvec(a, x, chunk) > c * (1.0 + FEAS_TOL)):
                raise RuntimeError("infeasible")
            objs.append(nv_objective_exact(x, mu, sigma, k_, h, v, chunk))
    return np.array(objs), x


# ---------------------------------------------------------------- instances (bench.py:102-137)
def uniform_range(stream, n, lo, hi):
    u = uniform01(stream, n)
    np.maximum(u, 2.0 ** -53, out=u)
    return lo + (hi - lo) * u


def gen_meanvar_instance(d, stream):
    mu = uniform_range(stream, d, -1.0, 1.0)
    sigma = uniform_range(stream, d, 0.0, 0.025)
    return mu, sigma


def gen_newsvendor_instance(n, stream):
    mu = uniform_range(stream, n, 20.0, 50.0)
    sigma = uniform_range(stream, n, 10.0, 20.0)
    k = uniform_range(stream, n, 1.0, 2.0)
    v = uniform_range(stream, n, 3.0, 5.0)
    h = uniform_range(stream, n, 0.5, 1.0)
    return dict(mu=mu, sigma=sigma, k=k, v=v, h=h, c=np.ones(n), budget=0.5 * float(np.sum(mu)))


# ---------------------------------------------------------------- task 3: logistic
def sample_indices(n, b, stream):
    """sampling.py:196-209 (partial Fisher-Yates, one uniform per index)."""
    u = uniform01(stream, b)
    idx = np.arange(n, dtype=np.int64)
    for i in range(b):
        j = i + int(u[i] * (n - i))
        idx[i], idx[j] = idx[j], idx[i]
    return idx[:b].copy()


def synth_classification(n_features, stream, n_rows=None):
    """sampling.py:229-265, generalised to n_rows (reference hard-codes 30*n)."""
    if n_rows is None:
        n_rows = 30 * n_features
    total = n_rows * n_features
    u = uniform01(stream, total)
    x = (u >= 0.5).astype(np.float64).reshape(n_rows, n_features)
    w_true = standard_normal(stream, n_features)
    scores = matvec(x, w_true)
    median = float(np.median(scores))
    labels = (scores > median).astype(np.float64)
    flip = sample_indices(n_rows, n_rows // 10, stream)
    labels[flip] = 1.0 - labels[flip]
    return x, labels, w_true


def _batch(x, z, indices):
    if indices is None:
        return x, z
    indices = np.asarray(indices)
    return x[indices], z[indices]


def logistic_loss(w, x, z, indices=None, chunk=CHUNK):
    """tasks.py:216-225."""
    xb, zb = _batch(x, z, indices)
    t = matvec(xb, w, chunk)
    terms = np.empty(t.size)
    lib().orc_logistic_loss_terms(_p(t), _p(np.ascontiguousarray(zb)), _p(terms), t.size)
    return vec_sum(terms, chunk) / t.size


def logistic_gradient(w, x, z, indices=None, chunk=CHUNK):
    """tasks.py:228-236."""
    xb, zb = _batch(x, z, indices)
    t = matvec(xb, w, chunk)
    c = sigmoid(t)
    return matvec_t(xb, c - zb, chunk) * (1.0 / t.size)


def logistic_hvp(w, v, x, z, indices=None, chunk=CHUNK):
    """tasks.py:239-253."""
    xb, _ = _batch(x, z, indices)
    t = matvec(xb, w, chunk)
    c = sigmoid(t)
    tv = matvec(xb, v, chunk)
    weighted = c * (1.0 - c) * tv
    return matvec_t(xb, weighted, chunk) * (1.0 / t.size)


def logistic_hessian_explicit(w, x, z):
    """Explicit Hessian oracle of tests/test_tasks.py:292-304 (not in sobench)."""
    t = matvec(x, w)
    c = sigmoid(t)
    return (x.T * (c * (1 - c))) @ x / x.shape[0]


def bfgs_rank2(h, s, u, coef_su, coef_ss):
    lib().orc_bfgs_rank2(_p(h), _p(_vec(s)), _p(_vec(u)), coef_su, coef_ss, h.shape[0])


def hessian_update(pairs, chunk=CHUNK):
    """sqn.py:75-110; pairs = [(s, y, curvature)] oldest first."""
    s_new, y_new, curv_new = pairs[-1]
    yy = dot(y_new, y_new, chunk)
    n = s_new.size
    h = np.zeros((n, n))
    np.fill_diagonal(h, curv_new / yy)
    for s, y, curv in pairs:
        rho = 1.0 / curv
        u = matvec(h, y, chunk)
        kappa = dot(y, u, chunk)
        bfgs_rank2(h, s, u, -rho, rho * rho * kappa + rho)
    return h


def sqn_run(x, z, *, pair_every, memory, beta, grad_batch, hess_batch, iterations, stream,
            chunk=CHUNK):
    """sqn.py:113-193 (SqnEngine.step + sqn_run) -> (objectives, final w)."""
    n_samples, n = x.shape
    w = np.zeros(n)
    wbar_accum = np.zeros(n)
    wbar_prev = None
    t = -1
    pairs = []
    inv_h = None
    objs = []
    for k in range(1, iterations + 1):
        batch = sample_indices(n_samples, grad_batch, stream)
        g = logistic_gradient(w, x, z, batch, chunk)
        wbar_accum = wbar_accum + w
        alpha = beta / k
        if k <= 2 * pair_every or inv_h is None:
            w = w - alpha * g
        else:
            w = w - alpha * matvec(inv_h, g, chunk)
        if k % pair_every == 0:
            t += 1
            wbar_new = wbar_accum * (1.0 / pair_every)
            if t > 0:
                hb = sample_indices(n_samples, hess_batch, stream)
                s = wbar_new - wbar_prev
                y = logistic_hvp(wbar_new, s, x, z, hb, chunk)
                curvature = dot(s, y, chunk)
                floor = CURVATURE_RTOL * math.sqrt(dot(s, s, chunk)) * math.sqrt(dot(y, y, chunk))
                if curvature > floor:
                    pairs.append((s, y, curvature))
                    pairs = pairs[-memory:]
                    inv_h = hessian_update(pairs, chunk)
            wbar_prev = wbar_new
            wbar_accum = np.zeros_like(wbar_accum)
        objs.append(logistic_loss(w, x, z, None, chunk))
    return np.array(objs), w


# ---------------------------------------------------------------- second-order solvers (no reference)
def newton_cg(x, z, *, iterations, cg_iters, chunk=CHUNK):
    """Newton-CG for the full-data logistic loss (BASELINE configs[2]; not in sobench).

    Restated with the reference's own building blocks (logistic_gradient /
    logistic_hvp / fixed-tree dot, tasks.py:228-253) so that the CUDA driver can be
    compared bit for bit:  p solves H p = -g by `cg_iters` CG steps from p = 0,
    then w <- w + p; the recorded objective is logistic_loss(w) after each step.
    """
    n = x.shape[1]
    w = np.zeros(n)
    objs = []
    for _ in range(iterations):
        g = logistic_gradient(w, x, z, None, chunk)
        p = np.zeros(n)
        r = -1.0 * g
        dd = r.copy()
        rr = dot(r, r, chunk)
        for _ in range(cg_iters):
            if rr == 0.0:
                break
            hd = logistic_hvp(w, dd, x, z, None, chunk)
            alpha = rr / dot(dd, hd, chunk)
            p = p + alpha * dd
            r = r - alpha * hd
            rr_new = dot(r, r, chunk)
            beta = rr_new / rr
            dd = r + beta * dd
            rr = rr_new
        w = w + p
        objs.append(logistic_loss(w, x, z, None, chunk))
    return np.array(objs), w


def newton_explicit(x, z, *, iterations, cg_iters, chunk=CHUNK):
    """Newton with the explicit Hessian H = (1/N) X^T diag(c(1-c)) X (tests/test_tasks.py:297-299
    oracle) and a CG solve on H (BASELINE configs[4]); H via numpy BLAS (any summation order)."""
    n = x.shape[1]
    w = np.zeros(n)
    objs = []
    for _ in range(iterations):
        g = logistic_gradient(w, x, z, None, chunk)
        h = logistic_hessian_explicit(w, x, z)
        p = np.zeros(n)
        r = -1.0 * g
        dd = r.copy()
        rr = float(r @ r)
        for _ in range(cg_iters):
            if rr == 0.0:
                break
            hd = h @ dd
            alpha = rr / float(dd @ hd)
            p = p + alpha * dd
            r = r - alpha * hd
            rr_new = float(r @ r)
            beta = rr_new / rr
            dd = r + beta * dd
            rr = rr_new
        w = w + p
        objs.append(logistic_loss(w, x, z, None, chunk))
    return np.array(objs), w


# ---------------------------------------------------------------- multi-PRNG
# Published-algorithm restatements (oracle/prng.c); parity with the reference's
# orphaned pkg/test_multi_prng_*.json fixtures is UNPINNED.
def philox4x32(ctr, key, nblocks):
    """uint32[4*nblocks]: Philox4x32-10 of counters ctr, ctr+1, ... (128-bit carry)."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.empty(4 * nblocks, dtype=np.uint32)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    lib().orc_philox4x32(c.ctypes.data_as(u32p), k.ctypes.data_as(u32p), nblocks,
                         out.ctypes.data_as(u32p))
    return out


def _gen64(fn, state, n):
    s = np.array(state, dtype=np.uint64)
    out = np.empty(n, dtype=np.uint64)
    fn(s.ctypes.data_as(_u64p), n, out.ctypes.data_as(_u64p))
    return out, s


def sfc64(state, n):
    """(outputs, new state) of SFC64 from state (a, b, c, counter)."""
    return _gen64(lib().orc_sfc64, state, n)


def xoshiro256pp(state, n):
    return _gen64(lib().orc_xoshiro256pp, state, n)


def xoshiro256pp_jump(state):
    s = np.array(state, dtype=np.uint64)
    lib().orc_xoshiro256pp_jump(s.ctypes.data_as(_u64p))
    return s


# ---------------------------------------------------------------- projected SGD
# No reference counterpart (sobench ships only Frank-Wolfe): restated from the
# standard exact algorithm (sort the breakpoints y_j / c_j; Held/Wolfe/Crowder,
# Duchi et al. 2008 for c = 1).  Checks csrc/project.cu and psgd.py by tolerance.
def project_budget(y, c=None, budget=1.0):
    """argmin ||x - y|| over {x >= 0, c.x <= budget}."""
    y = _vec(y)
    c = np.ones(y.size) if c is None else _vec(c)
    x0 = np.maximum(y, 0.0)
    if c @ x0 <= budget:
        return x0
    t = y / c
    order = np.argsort(-t, kind="stable")
    cy = np.cumsum(c[order] * y[order])
    cc = np.cumsum(c[order] ** 2)
    theta = (cy - budget) / cc
    ok = np.nonzero(theta < t[order])[0]
    th = theta[ok[-1]]
    return np.maximum(y - th * c, 0.0)


def psgd_run_meanvar(mu, sigma, epochs, inner_iters, n_samples, stream, step0=1.0, chunk=CHUNK):
    d = mu.size
    w = np.zeros(d)
    objs = []
    t = 0
    for _ in range(epochs):
        x = sample_returns_diag(mu, sigma, n_samples, stream)
        mean, xc = build_sample_set(x, chunk)
        for _ in range(inner_iters):
            g = mv_gradient(w, mean, xc, chunk)
            w = project_budget(w - (step0 / math.sqrt(t + 1)) * g, None, 1.0)
            objs.append(mv_objective(w, mean, xc, chunk))
            t += 1
    return np.array(objs), w
