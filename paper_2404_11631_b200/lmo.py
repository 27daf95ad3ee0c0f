"""Linear minimization oracles (mirror of sobench/lmo.py) on the device.

``lmo_simplex_slack`` / ``lmo_single_budget`` run a deterministic first-argmin
kernel (csrc/fw.cu).  ``lmo_general`` -- the reference's dense Bland simplex for
small multi-resource polytopes (lmo.py:92-160) -- runs the same pivots on the
device in one CTA (csrc/lp.cu).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import empty, like_input, vec_dev
from ._tensors import mat_dev, to_dev
from .errors import DimensionMismatch, InvalidConstraint, InvalidGradient, SolverStall


@dataclass
class SimplexSlackSet:
    """{w : sum(w) <= 1, w >= 0} (lmo.py:20-24)."""

    dimension: int


@dataclass
class PolytopeSet:
    """{s : A s <= C, s >= 0} with strictly positive A and C (lmo.py:27-52)."""

    A: np.ndarray
    C: np.ndarray

    def __post_init__(self):
        self.A = np.ascontiguousarray(self.A, dtype=np.float64)
        self.C = np.ascontiguousarray(self.C, dtype=np.float64)
        if self.A.ndim != 2:
            raise DimensionMismatch(f"expected 2-D matrix, got shape {self.A.shape}")
        if self.C.ndim != 1:
            raise DimensionMismatch(f"expected 1-D vector, got shape {self.C.shape}")
        if self.A.shape[0] != self.C.size:
            raise DimensionMismatch("constraint rows != len(C)")
        if not np.all(self.A > 0):
            raise InvalidConstraint("technology matrix entries must be strictly positive")
        if not np.all(self.C > 0):
            raise InvalidConstraint("budget levels must be strictly positive")
        self._dev = None

    @property
    def n_resources(self) -> int:
        return self.A.shape[0]

    @property
    def n_products(self) -> int:
        return self.A.shape[1]

    def device(self):
        """(A, C) on the device, uploaded once."""
        if self._dev is None:
            self._dev = (mat_dev(self.A), to_dev(self.C))
        return self._dev


def lmo_general_device(g: torch.Tensor, polytope: PolytopeSet, max_iters: int | None = None,
                       out=None) -> torch.Tensor:
    m, n = polytope.A.shape
    if g.numel() != n:
        raise DimensionMismatch(f"gradient length {g.numel()} != products {n}")
    cap = max_iters if max_iters is not None else 10 * (n + m)
    a, c = polytope.device()
    out = empty(n) if out is None else out
    st = _status_tensor()
    _lib.call("simopt_lmo_general", _lib.stream_ptr(), _lib.ptr(a), _lib.ptr(c), m, n, _lib.ptr(g),
              int(cap), _lib.ptr(out), _lib.ptr(st))
    code = int(st.item())
    if code == 5:
        raise InvalidGradient("gradient contains NaN")
    if code == 7:
        raise SolverStall("LP unbounded; polytope invariants violated")
    if code == -7:
        raise SolverStall(f"simplex exceeded {cap} iterations")
    return out


def lmo_general(g, polytope: PolytopeSet, max_iters: int | None = None):
    """argmin of s.g over {A s <= C, s >= 0} by primal simplex (lmo.py:92-160)."""
    return like_input(g, lmo_general_device(vec_dev(g), polytope, max_iters))


def _status_tensor():
    return torch.zeros(1, dtype=torch.int32, device="cuda")


def _raise_status(status: torch.Tensor):
    if int(status.item()) != 0:
        raise InvalidGradient("gradient contains NaN")


def lmo_simplex_slack_device(g: torch.Tensor, out=None, status=None) -> torch.Tensor:
    out = empty(g.numel()) if out is None else out
    st = _status_tensor() if status is None else status
    _lib.call("simopt_lmo_simplex_slack", _lib.stream_ptr(), _lib.ptr(g), g.numel(), _lib.ptr(out),
              _lib.ptr(st))
    if status is None:
        _raise_status(st)
    return out


def lmo_simplex_slack(g):
    """argmin over the simplex-with-slack of s.g: a basis vector or zero (lmo.py:56-65)."""
    return like_input(g, lmo_simplex_slack_device(vec_dev(g)))


def lmo_single_budget_device(g: torch.Tensor, c: torch.Tensor, budget: float, out=None,
                             status=None) -> torch.Tensor:
    out = empty(g.numel()) if out is None else out
    st = _status_tensor() if status is None else status
    _lib.call("simopt_lmo_single_budget", _lib.stream_ptr(), _lib.ptr(g), _lib.ptr(c), float(budget),
              g.numel(), _lib.ptr(out), _lib.ptr(st))
    if status is None:
        _raise_status(st)
    return out


def lmo_single_budget(g, c, budget: float):
    """argmin of s.g over {c.s <= budget, s >= 0} (lmo.py:68-89)."""
    gd, cd = vec_dev(g), vec_dev(c)
    if gd.numel() != cd.numel():
        raise DimensionMismatch("gradient and cost lengths differ")
    if not bool((cd > 0).all()):
        raise InvalidConstraint("resource costs must be strictly positive")
    if not budget > 0:
        raise InvalidConstraint("budget must be strictly positive")
    return like_input(g, lmo_single_budget_device(gd, cd, budget))
