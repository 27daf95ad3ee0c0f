"""Benchmark instance generators (mirror of sobench/bench.py:102-141).

Draws come from the device Philox stream (bit-identical to the reference);
the d-vector arithmetic is the reference's own numpy expression.
"""
from __future__ import annotations

import numpy as np

from .errors import ConfigurationError
from .sampling import GaussianSpec, RngStream, uniform01


def uniform_range(stream: RngStream, n: int, lo: float, hi: float) -> np.ndarray:
    """bench.py:102-107: lo + (hi - lo) * max(u, 2^-53)."""
    u = uniform01(stream, n)
    np.maximum(u, 2.0 ** -53, out=u)
    return lo + (hi - lo) * u


def gen_meanvar_instance(d: int, stream: RngStream):
    """mu ~ U(-1,1)^d, sigma ~ U(0, 0.025)^d, diagonal covariance (bench.py:110-116)."""
    from .tasks import MeanVarTask
    if d < 2:
        raise ConfigurationError("need at least 2 assets")
    mu = uniform_range(stream, d, -1.0, 1.0)
    sigma = uniform_range(stream, d, 0.0, 0.025)
    return MeanVarTask(spec=GaussianSpec(mean=mu, diag_std=sigma))


def gen_newsvendor_instance(n: int, stream: RngStream):
    """bench.py:119-137: mu~U(20,50), sigma~U(10,20), k~U(1,2), v~U(3,5), h~U(0.5,1), C=0.5*sum(mu)."""
    from .tasks import NewsvendorTask
    if n < 1:
        raise ConfigurationError("need at least 1 product")
    mu = uniform_range(stream, n, 20.0, 50.0)
    sigma = uniform_range(stream, n, 10.0, 20.0)
    k = uniform_range(stream, n, 1.0, 2.0)
    v = uniform_range(stream, n, 3.0, 5.0)
    h = uniform_range(stream, n, 0.5, 1.0)
    return NewsvendorTask(unit_cost=k, holding_cost=h, selling_value=v, demand_mean=mu,
                          demand_std=sigma, budget_costs=np.ones(n), budget=0.5 * float(np.sum(mu)))
