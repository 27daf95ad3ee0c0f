"""The "cuda" compute backend: sobench's Backend surface on sm_100a kernels.

Mirrors sobench/backend.py:50-213.  Every reduction follows the reference's
fixed tree (chunk-local sequential sums, pairwise fold in index order), so
``CudaBackend`` is bit-identical to ``SequentialBackend``/``ParallelBackend``
-- the same contract the reference enforces between its two CPU backends
(backend.py:1-15).  Inputs may be host arrays (copied in, result copied out:
correct but PCIe-bound) or CUDA tensors (result stays on the device).

The kind string is "cuda", never "gpu": the reference's own test suite
asserts ``make_backend("gpu")`` raises (tests/test_backend.py:214-216).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import empty, is_tensor, like_input, mat_dev, to_dev, vec_dev
from .errors import ConfigurationError, DimensionMismatch

DEFAULT_CHUNK = 4096
MAP_KERNELS = ("sigmoid", "negate", "exp")
_MAP_IDS = {"sigmoid": 0, "negate": 1, "exp": 2}


class CudaBackend:
    """Fixed-tree kernels on the current CUDA device (backend.py:50-164 surface)."""

    kind = "cuda"

    def __init__(self, chunk_size: int = DEFAULT_CHUNK, workers: int | None = None):
        if chunk_size < 1:
            raise ConfigurationError(f"chunk_size must be >= 1, got {chunk_size}")
        self.chunk_size = int(chunk_size)
        self.workers = 1  # accepted for API compatibility; parallelism is the GPU's
        _lib.load()

    # -- range scheduling (backend.py:68-76) ----------------------------------
    def run_blocks(self, n_units: int, fn, work_per_unit: int = 1):
        """The reference API's host-callback hook (backend.py:68-76).

        Reference task code passes closures over its numba CPU kernels here.  The cuda
        backend never runs them: that would be a silent CPU fallback.  The reference's
        task, sampling and SQN functions are routed to the device implementations
        instead (``sobench_plugin.install()``); anything else raises.
        """
        raise ConfigurationError(
            "the cuda backend does not run host callbacks (backend.run_blocks): call this "
            "package's device implementation, or install paper_2404_11631_b200.sobench_plugin "
            "so sobench's task functions route to it")

    # -- reductions (backend.py:80-141) ----------------------------------------
    def dot_device(self, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None):
        if x.numel() != y.numel():
            raise DimensionMismatch(f"dot: lengths {x.numel()} != {y.numel()}")
        out = empty(1) if out is None else out
        _lib.call("simopt_dot", _lib.stream_ptr(), _lib.ptr(x), _lib.ptr(y), x.numel(),
                  self.chunk_size, _lib.ptr(out))
        return out

    def dot(self, x, y):
        xd, yd = vec_dev(x), vec_dev(y)
        r = self.dot_device(xd, yd)
        return r[0] if (is_tensor(x) and is_tensor(y)) else float(r.item())

    def vec_sum_device(self, x: torch.Tensor, out: torch.Tensor | None = None):
        out = empty(1) if out is None else out
        _lib.call("simopt_vec_sum", _lib.stream_ptr(), _lib.ptr(x), x.numel(), self.chunk_size,
                  _lib.ptr(out))
        return out

    def vec_sum(self, x):
        r = self.vec_sum_device(vec_dev(x))
        return r[0] if is_tensor(x) else float(r.item())

    def matvec_device(self, a, x, out=None, rows_idx=None, center=None):
        """out[r] = tree-dot(a[row(r)] - center, x); row(r) = rows_idx[r] if given."""
        rows = a.shape[0] if rows_idx is None else rows_idx.numel()
        cols = a.shape[1]
        if cols != x.numel():
            raise DimensionMismatch(f"matvec: {tuple(a.shape)} @ ({x.numel()},)")
        out = empty(rows) if out is None else out
        _lib.call("simopt_matvec", _lib.stream_ptr(), _lib.ptr(a), a.shape[0], cols,
                  _lib.ptr(rows_idx), rows, _lib.ptr(center), _lib.ptr(x), self.chunk_size,
                  _lib.ptr(out))
        return out

    def matvec(self, a, x):
        return like_input(a, self.matvec_device(mat_dev(a), vec_dev(x)))

    def matvec_t_device(self, a, x, out=None, rows_idx=None, center=None):
        rows = a.shape[0] if rows_idx is None else rows_idx.numel()
        cols = a.shape[1]
        if rows != x.numel():
            raise DimensionMismatch(f"matvec_t: {tuple(a.shape)}^T @ ({x.numel()},)")
        out = empty(cols) if out is None else out
        _lib.call("simopt_matvec_t", _lib.stream_ptr(), _lib.ptr(a), a.shape[0], cols,
                  _lib.ptr(rows_idx), rows, _lib.ptr(center), _lib.ptr(x), self.chunk_size,
                  _lib.ptr(out))
        return out

    def matvec_t(self, a, x):
        return like_input(a, self.matvec_t_device(mat_dev(a), vec_dev(x)))

    # -- elementwise (backend.py:127-164) -------------------------------------
    def axpy_device(self, alpha, x, y, out=None):
        if x.numel() != y.numel():
            raise DimensionMismatch(f"axpy: lengths {x.numel()} != {y.numel()}")
        out = empty(x.numel()) if out is None else out
        _lib.call("simopt_axpy", _lib.stream_ptr(), float(alpha), _lib.ptr(x), _lib.ptr(y),
                  x.numel(), _lib.ptr(out))
        return out

    def axpy(self, alpha: float, x, y):
        return like_input(x, self.axpy_device(alpha, vec_dev(x), vec_dev(y)))

    def map_kernel_device(self, kernel: str, x, out=None):
        if kernel not in _MAP_IDS:
            raise ConfigurationError(f"unknown map kernel {kernel!r}")
        out = empty(x.numel()) if out is None else out
        _lib.call("simopt_map_kernel", _lib.stream_ptr(), _MAP_IDS[kernel], _lib.ptr(x),
                  x.numel(), _lib.ptr(out))
        return out

    def map_kernel(self, kernel: str, x):
        if kernel not in _MAP_IDS:
            raise ConfigurationError(f"unknown map kernel {kernel!r}")
        return like_input(x, self.map_kernel_device(kernel, vec_dev(x)))


def make_backend(kind: str, chunk_size: int = DEFAULT_CHUNK, workers: int | None = None) -> CudaBackend:
    """Build a backend from its config-string name (backend.py:207-213).

    Only "cuda" exists in this package: the reference's "sequential" and
    "parallel" CPU backends are not re-implemented (there is no CPU path).
    """
    if kind == "cuda":
        return CudaBackend(chunk_size, workers)
    raise ConfigurationError(f"unknown backend {kind!r} (expected 'cuda')")
