"""Single-pass fused streaming evaluations (csrc/fused.cu, ABI simopt_fused_rows).

The reference evaluates every big pass as ``matvec`` then ``matvec_t`` over the
same matrix (mean-variance gradient tasks.py:78-85, logistic gradient
tasks.py:228-236, logistic HVP tasks.py:239-253): two reads of X.  The fused
kernel reads X once.  Its summation order is not the reference's fixed tree
(the exact-tree kernels stay the parity mode), so results agree to ~1e-15
relative -- inside the north star's 1e-10 gradient and 1e-8 trajectory gates.
"""
from __future__ import annotations

import torch

from . import _lib

MV, LR_GRAD, LR_HVP = 0, 1, 2


def fused_rows(mode: int, x: torch.Tensor, v: torch.Tensor, *, center=None, rowaux=None,
               col_scale: float = 1.0, col_out=None, scalar_out=None, t_out=None, dw_out=None,
               accumulate: bool = True, raw: bool = False):
    """One read of x (N x d, fp64, row-major, on the device); see include/simopt_b200.h."""
    n, d = x.shape
    P = _lib.ptr
    _lib.call("simopt_fused_rows", _lib.stream_ptr(), int(mode), P(x), n, d, P(v), P(center),
              P(rowaux), float(col_scale), 1 if accumulate else 0, 1 if raw else 0, P(t_out), P(dw_out),
              P(col_out), P(scalar_out))
    return col_out


def fused_rows_bits(mode: int, bits: torch.Tensor, d: int, v: torch.Tensor, *, rowaux,
                    col_scale: float = 1.0, col_out=None, scalar_out=None, t_out=None, dw_out=None,
                    accumulate: bool = True, raw: bool = False):
    """The logistic passes on bit-packed features (N x ceil(d/64) words)."""
    P = _lib.ptr
    _lib.call("simopt_fused_rows_bits", _lib.stream_ptr(), int(mode), P(bits), bits.shape[0], d,
              P(v), P(rowaux), float(col_scale), 1 if accumulate else 0, 1 if raw else 0, P(t_out),
              P(dw_out), P(col_out), P(scalar_out))
    return col_out
