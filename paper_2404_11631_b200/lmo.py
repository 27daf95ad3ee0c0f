"""Linear minimization oracles (mirror of sobench/lmo.py) on the device.

``lmo_simplex_slack`` / ``lmo_single_budget`` run a deterministic first-argmin
kernel (csrc/fw.cu).  ``lmo_general`` -- the reference's dense Bland simplex for
small multi-resource polytopes (lmo.py:92-160) -- is out of scope for this
package (not on any benchmark configuration).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import empty, like_input, vec_dev
from .errors import DimensionMismatch, InvalidConstraint, InvalidGradient


@dataclass
class SimplexSlackSet:
    """{w : sum(w) <= 1, w >= 0} (lmo.py:20-24)."""

    dimension: int


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
