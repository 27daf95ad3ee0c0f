"""Second-order Newton solvers for the classification task (BASELINE.json configs[2], [4]).

The reference package only ships SQN (sobench/sqn.py); these drivers are the
north star's "CG/Cholesky Newton step" built from the reference's own building
blocks, with CPU restatements in oracle/oracle.py (newton_cg / newton_explicit):

* ``newton_cg`` -- full-data gradient (tasks.py:228-236) and CG on
  Hessian-vector products (tasks.py:239-253).  The HVP weights c(1-c) depend on
  w only, so they are formed once per Newton iteration and reused by every CG
  product (same IEEE values as recomputing them); ``X w`` from the recorded
  loss is reused by the next gradient.  All reductions use the exact tree, so
  the trajectory is bit-identical to the oracle.
* ``newton_explicit`` -- explicit H = (1/N) X^T diag(c(1-c)) X on the FP64 tensor
  pipe (csrc/hessian.cu) and a CG solve on H; parity to the numpy-BLAS oracle
  is within tolerance (rtol 1e-10 on H, 1e-8 on the trajectory).

Every scalar of the CG recurrences stays on the device (simopt_cg_step1/2), so an
iteration is one uninterrupted stream of kernels; the objective trace is read
once at the end.

``fused=True`` (the default) evaluates each gradient+loss and each HVP with the
single-pass kernel of csrc/fused.cu -- one read of X instead of two, k_CG + 1
reads per Newton iteration (SURVEY 8d's algorithmic bytes) -- in a fast
summation order (trajectory within 1e-8 of the oracle).  ``fused=False`` keeps
the exact fixed tree and the bit-identical trajectory.
"""
from __future__ import annotations

import os

import torch

from . import _lib
from ._tensors import F64, empty, to_host
from .fused import LR_GRAD, LR_HVP, PeerReducer, fused_rows, fused_rows_bits
from .records import RunRecord, TraceBuilder
from .tasks import x_matvec, x_matvec_t

_SCALE, _MUL = 3, 4


def _vop(op, alpha, x, y, out):
    _lib.call("simopt_vec_op", _lib.stream_ptr(), op, float(alpha), _lib.ptr(x), _lib.ptr(y),
              x.numel(), _lib.ptr(out))
    return out


class _Logistic:
    """Per-run buffers for the full-data logistic passes."""

    def __init__(self, data, backend, exchange="peer"):
        self.data, self.b = data, backend
        self.N, self.d = data.n_samples, data.n_features   # N: global rows
        self.shard = getattr(data, "shard", None)
        nl = max(data.local_rows, 1)                        # this rank's rows
        self.nl = data.local_rows
        self.t = empty(nl)       # X w
        self.r = empty(nl)       # residual / hvp weights scratch
        self.dw = empty(nl)      # c (1 - c)
        self.tv = empty(nl)
        self.gt = empty(self.d)
        self.buf = empty(self.d + 1)  # [column sums | side sum] allreduced across shards
        self.ones = torch.ones(nl, dtype=F64, device="cuda")
        # sample-sharded fused passes: cross-rank sums inside the finish kernel over peer
        # memory (None -> raw partials + NCCL allreduce)
        self.pr = (PeerReducer.get(self.shard, self.d)
                   if self.shard is not None and exchange == "peer" else None)

    def _pass(self, mode, v, rowaux, **kw):
        """One fused read of this rank's rows (bit-packed features when available)."""
        if self.data.packed:
            return fused_rows_bits(mode, self.data.bits, self.d, v, rowaux=rowaux, **kw)
        return fused_rows(mode, self.data.features, v, rowaux=rowaux, **kw)

    def _col_sums(self, v, out):
        """Fixed-tree X^T v over all rows (gathered chunk partials when sharded)."""
        if self.shard is None:
            return x_matvec_t(self.data, self.b, v[:self.nl], out=out)
        from .tasks import sharded_matvec_t
        return sharded_matvec_t(self.shard, self.data.features, v[:self.nl], self.N,
                                self.b.chunk_size, out=out)

    def _scale(self, src, out):
        _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(src), 1.0 / self.N, None,
                  self.d, _lib.ptr(out))
        return out

    def xw(self, w):
        if self.nl:
            x_matvec(self.data, self.b, w, out=self.t[:self.nl])
        return self.t

    def gradient_from_t(self, out):
        """(1/N) X^T (sigmoid(t) - z) given t = X w (tasks.py:228-236)."""
        if self.nl:
            _lib.call("simopt_logistic_resid", _lib.stream_ptr(), _lib.ptr(self.t),
                      _lib.ptr(self.data.labels), None, self.nl, _lib.ptr(self.r))
        self._col_sums(self.r, self.gt)
        return self._scale(self.gt, out)

    def hvp_weights_from_t(self):
        """c (1 - c) -- identical to the (c*(1-c)) factor of tasks.py:252."""
        if self.nl:
            _lib.call("simopt_logistic_hvp_weights", _lib.stream_ptr(), _lib.ptr(self.t),
                      _lib.ptr(self.ones), self.nl, _lib.ptr(self.dw))

    def hvp(self, v, out):
        """(1/N) X^T ((c(1-c)) * (X v))."""
        if self.nl:
            x_matvec(self.data, self.b, v, out=self.tv[:self.nl])
            _vop(_MUL, 0.0, self.dw, self.tv, self.r)
        self._col_sums(self.r, self.gt)
        return self._scale(self.gt, out)

    def fused_gradient(self, w, g_out, loss_sum_out):
        """One pass: g = (1/N) X^T (sigmoid(Xw) - z), sum of loss terms, c(1-c) for the HVPs."""
        if self.shard is None or self.pr is not None:
            self._pass(LR_GRAD, w, self.data.labels, col_scale=1.0 / self.N, col_out=g_out,
                       scalar_out=loss_sum_out, dw_out=self.dw, peer=self.pr)
            return
        # per-shard raw sums, one allreduce of d+1 doubles
        self._pass(LR_GRAD, w, self.data.labels, col_out=self.buf[:self.d],
                   scalar_out=self.buf[self.d:], dw_out=self.dw, raw=True)
        self.shard.allreduce_(self.buf)
        self._scale(self.buf, g_out)
        loss_sum_out[:1].copy_(self.buf[self.d:])

    def fused_hvp(self, v, out):
        """One pass: (1/N) X^T ((c(1-c)) * (X v))."""
        if self.shard is None or self.pr is not None:
            return self._pass(LR_HVP, v, self.dw, col_scale=1.0 / self.N, col_out=out, peer=self.pr)
        self._pass(LR_HVP, v, self.dw, col_out=self.buf[:self.d], raw=True)
        self.shard.allreduce_(self.buf[:self.d])
        return self._scale(self.buf, out)

    def loss_sum_from_t(self, out):
        if self.nl:
            _lib.call("simopt_logistic_loss_terms", _lib.stream_ptr(), _lib.ptr(self.t),
                      _lib.ptr(self.data.labels), None, self.nl, _lib.ptr(self.r))
        if self.shard is None:
            return self.b.vec_sum_device(self.r, out=out)
        from .tasks import sharded_matvec_t
        # exact sum over shards: partials of the (n x 1) column r against ones (r * 1.0 == r)
        return sharded_matvec_t(self.shard, self.r[:self.nl].view(-1, 1), self.ones[:self.nl],
                                self.N, self.b.chunk_size, out=out[:1])


def _cg(apply, g, n, cg_iters, dot, p):
    """p solves A p = -g by cg_iters CG steps from p = 0 (oracle.newton_cg inner loop)."""
    p.zero_()
    r = empty(n)
    _vop(_SCALE, -1.0, g, g, r)                  # r = -1.0 * g
    dd = r.clone()
    hd = empty(n)
    sc = torch.empty(3, dtype=F64, device="cuda")  # rr (ping), dHd, rr (pong)
    dot(r, r, sc[0:])
    for i in range(cg_iters):
        # rr and rr_new swap slots each step (rr <- rr_new without a copy).  Once rr == 0
        # the steps are no-ops, r stays put and every later r.r is 0 again: the oracle's
        # `break`
        rr, rr_new = (sc[0:], sc[2:]) if i % 2 == 0 else (sc[2:], sc[0:])
        apply(dd, hd)
        dot(dd, hd, sc[1:])
        _lib.call("simopt_cg_step1", _lib.stream_ptr(), _lib.ptr(p), _lib.ptr(r), _lib.ptr(dd),
                  _lib.ptr(hd), _lib.ptr(rr), _lib.ptr(sc[1:]), n)
        dot(r, r, rr_new)
        _lib.call("simopt_cg_step2", _lib.stream_ptr(), _lib.ptr(dd), _lib.ptr(r), _lib.ptr(rr_new),
                  _lib.ptr(rr), n)
    return p


def _run(task, iterations, backend, step, label, fused=False, exchange="peer", on_iteration=None):
    data = task.data
    L = _Logistic(data, backend, exchange if fused else "nccl")
    n = L.d
    w = torch.zeros(n, dtype=F64, device="cuda")
    g = empty(n)
    p = empty(n)
    sums = empty(iterations)
    stamps = torch.zeros(iterations + 1, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    _lib.check(lib.simopt_timestamp(_lib.stream_ptr(), _lib.ptr(stamps[iterations:])))
    if fused and n <= 65536 and os.environ.get("SIMOPT_CG_TREE") != "1":  # one-CTA CG scalars
        def dot(x, y, out):
            _lib.call("simopt_dot_fast", _lib.stream_ptr(), _lib.ptr(x), _lib.ptr(y), x.numel(),
                      _lib.ptr(out))
            return out
    else:
        dot = lambda x, y, out: backend.dot_device(x, y, out=out)  # noqa: E731
    if fused:
        loss0 = empty(1)
        L.fused_gradient(w, g, loss0)
    else:
        L.xw(w)
    for it in range(iterations):
        if not fused:
            L.gradient_from_t(g)
            L.hvp_weights_from_t()
        step(L, g, p, dot)
        _lib.call("simopt_vec_op", _lib.stream_ptr(), 1, 0.0, _lib.ptr(w), _lib.ptr(p), n,
                  _lib.ptr(w))                    # w = w + p
        if fused:  # loss at the new iterate + the next gradient and HVP weights, one pass
            L.fused_gradient(w, g, sums[it:])
        else:
            L.xw(w)                               # shared by the loss and the next gradient
            L.loss_sum_from_t(sums[it:])
        _lib.check(lib.simopt_timestamp(_lib.stream_ptr(), _lib.ptr(stamps[it:])))
        if on_iteration is not None:  # e.g. bench.py records a CUDA event per iteration
            on_iteration(it)
    if L.pr is not None:
        L.pr.check()
    trace = TraceBuilder()
    vals, ts = to_host(sums), to_host(stamps)
    for it in range(iterations):
        trace.append(it + 1, float(vals[it]) / L.N, int(ts[it]) - int(ts[iterations]))
    return trace.build(label, n, backend.kind, 0, 0, to_host(w))


def newton_cg(task, iterations: int, cg_iters: int, backend, fused: bool = True,
              exchange: str = "peer", on_iteration=None) -> RunRecord:
    """Newton-CG on the full-data logistic loss (BASELINE.json configs[2]).
    on_iteration(it): called after iteration it is enqueued (host side)."""
    def step(L, g, p, dot):
        _cg(L.fused_hvp if fused else L.hvp, g, L.d, cg_iters, dot, p)
    return _run(task, iterations, backend, step, "classification-newton-cg", fused, exchange,
                on_iteration)


def logistic_hessian_device(data, dw, out=None, method: str = "auto") -> torch.Tensor:
    """H = (1/N) X^T diag(dw) X (tests/test_tasks.py:297-299 oracle, rtol 1e-10).

    method: "dmma" -- FP64 tensor pipe (csrc/hessian.cu; fp64 or bit-packed X);
    "i8" / "tc" / "tma" -- bit-packed binary X only: exact 5-limb split of dw on the
    integer tensor cores, warp-level IMMA ("i8") or tcgen05 with TMEM accumulators, its
    operands by cp.async ("tc") or TMA ("tma") (csrc/hessian_i8.cu); "auto" = "tma" for
    bit-packed data, else "dmma".  The limb methods quantise dw with an exponent taken
    from max(dw) and add exact-residual refinement passes when the worst-case bound
    2^-40 max(dw)/mean(dw) exceeds 1e-11 (`logistic_hessian_device.last_passes`).
    Row-sharded data: each rank's (1/N_loc) X_loc^T D X_loc is weighted by N_loc/N and
    summed over ranks with one allreduce of the d x d matrix."""
    d = data.n_features
    out = torch.empty(d, d, dtype=F64, device="cuda") if out is None else out
    nl = data.local_rows
    shard = getattr(data, "shard", None)
    if method == "auto":
        method = "tma" if data.packed else "dmma"
    if nl and method in ("i8", "tc", "tma", "pair"):
        xt, np_ = data.feature_major_u8()
        limbs = getattr(data, "_limbs", None)
        if limbs is None or limbs.numel() != 5 * np_:
            limbs = data._limbs = torch.empty(5 * np_, dtype=torch.uint8, device="cuda")
        fn = {"tc": "simopt_logistic_xtdx_tc", "tma": "simopt_logistic_xtdx_tma",
              "pair": "simopt_logistic_xtdx_pair", "i8": "simopt_logistic_xtdx_i8"}[method]
        _lib.call(fn,
                  _lib.stream_ptr(), _lib.ptr(xt), np_, nl, d, _lib.ptr(dw), _lib.ptr(limbs),
                  _lib.ptr(out))
        # 1, or 3 when the precision guard refined a wide spread of dw (csrc/hessian_i8.cu)
        logistic_hessian_device.last_passes = int(_lib.load().simopt_xtdx_last_passes())
    elif nl and data.packed:
        _lib.call("simopt_logistic_xtdx_bits", _lib.stream_ptr(), _lib.ptr(data.bits), _lib.ptr(dw),
                  nl, d, _lib.ptr(out))
    elif nl:
        _lib.call("simopt_logistic_xtdx", _lib.stream_ptr(), _lib.ptr(data.features), _lib.ptr(dw),
                  nl, d, _lib.ptr(out))
    else:
        out.zero_()
    if shard is not None:
        if nl:
            out.mul_(nl / data.n_samples)
        shard.allreduce_(out)
    return out


def newton_explicit(task, iterations: int, cg_iters: int, backend, fused: bool = True,
                    hessian: str = "auto", exchange: str = "peer", on_iteration=None) -> RunRecord:
    """Newton with the explicit X^T D X Hessian and a CG solve (BASELINE.json configs[4])."""
    d = task.data.n_features
    H = torch.empty(d, d, dtype=F64, device="cuda")

    def step(L, g, p, dot):
        logistic_hessian_device(L.data, L.dw, out=H, method=hessian)
        _cg(lambda v, out: backend.matvec_device(H, v, out=out), g, d, cg_iters, dot, p)
    return _run(task, iterations, backend, step, "classification-newton-explicit", fused, exchange,
                on_iteration)


logistic_hessian_device.last_passes = 0  # set by the limb methods
