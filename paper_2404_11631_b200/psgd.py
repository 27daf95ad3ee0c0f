"""Projected stochastic gradient driver (BASELINE.json configs[0]: "first-order
(Frank-Wolfe/projected SGD)").

The reference ships only Frank-Wolfe (sobench/frank_wolfe.py); this driver keeps
fw_run's contract -- K resampling epochs x M inner steps, the recorded objective
is the new iterate's under the epoch's samples, RunAborted carries the partial
trace -- and replaces the LMO + convex-combination update by
    w <- P(w - alpha_t g),   alpha_t = step0 / sqrt(t + 1)  (t = global step),
with P the Euclidean projection onto the problem's feasible set
(csrc/project.cu: simplex-with-slack for mean-variance, the single budget
polytope for the newsvendor).  Parity: oracle/oracle.py psgd_run_meanvar
(exact sort-based projection), trajectories within 1e-8.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import F64, empty, to_host, vec_dev
from .errors import ConfigurationError, InvalidConstraint, InvalidGradient, RunAborted
from .records import RunRecord, TraceBuilder
from .sampling import RngStream


@dataclass
class PsgdConfig:
    epochs: int
    inner_iters: int
    sample_size: int
    stream: RngStream
    step0: float = 1.0

    def __post_init__(self):
        if self.epochs < 1 or self.inner_iters < 1 or self.sample_size < 1:
            raise ConfigurationError("epochs, inner_iters and sample_size must be >= 1")
        if not self.step0 > 0:
            raise ConfigurationError("step0 must be > 0")


def psgd_step_size(step0: float, t: int) -> float:
    return step0 / math.sqrt(t + 1)


def project_budget(y, c=None, budget: float = 1.0, out=None) -> torch.Tensor:
    """Euclidean projection onto {x >= 0, c.x <= budget} (c None: all ones)."""
    yd = vec_dev(y)
    out = empty(yd.numel()) if out is None else out
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    cd = None if c is None else vec_dev(c)
    _lib.call("simopt_project_budget", _lib.stream_ptr(), _lib.ptr(yd), _lib.ptr(cd), float(budget),
              yd.numel(), _lib.ptr(out), _lib.ptr(st))
    if int(st.item()):
        raise InvalidGradient("projection input contains NaN")
    return out


def project_box(y, lo: float, hi: float, out=None) -> torch.Tensor:
    yd = vec_dev(y)
    out = empty(yd.numel()) if out is None else out
    _lib.call("simopt_project_box", _lib.stream_ptr(), _lib.ptr(yd), float(lo), float(hi),
              yd.numel(), _lib.ptr(out))
    return out


def psgd_run(problem, config: PsgdConfig, backend, *, task_label: str | None = None,
             size: int | None = None, rep: int = 0) -> RunRecord:
    """K*M projected stochastic gradient steps on a problem exposing .project(y)."""
    label = task_label or getattr(problem, "name", "task")
    dim = size if size is not None else problem.dimension
    trace = TraceBuilder()
    w = torch.zeros(problem.dimension, dtype=F64, device="cuda")
    y = empty(problem.dimension)
    start = time.perf_counter_ns()
    try:
        t = 0
        for k in range(config.epochs):
            problem.resample(config.stream, config.sample_size)
            for _ in range(config.inner_iters):
                g = problem.gradient(w)
                _lib.call("simopt_axpy", _lib.stream_ptr(), -psgd_step_size(config.step0, t),
                          _lib.ptr(g), _lib.ptr(w), w.numel(), _lib.ptr(y))
                w = problem.project(y)
                if not problem.check_feasible(w):
                    raise InvalidConstraint(f"iterate infeasible at step {t + 1}")
                f = problem.objective(w)
                t += 1
                trace.append(t, f, time.perf_counter_ns() - start)
    except Exception as exc:
        partial = trace.build(label, dim, backend.kind, rep, config.stream.seed, to_host(w))
        raise RunAborted(f"projected SGD run failed at step {len(trace) + 1}: {exc}", partial) from exc
    return trace.build(label, dim, backend.kind, rep, config.stream.seed, to_host(w))
