"""Host/device conversion helpers (device = the current CUDA device, float64)."""
from __future__ import annotations

import numpy as np
import torch

from .errors import DimensionMismatch

F64 = torch.float64


def device():
    return torch.device("cuda", torch.cuda.current_device())


def is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_dev(x, dtype=F64) -> torch.Tensor:
    """C-contiguous device tensor (copies host data; no copy for matching device tensors)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.device.type != "cuda":
            t = t.to(device())
        if t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    a = np.ascontiguousarray(x, dtype=np.float64 if dtype == F64 else np.int64)
    return torch.from_numpy(a).to(device(), non_blocking=False)


def vec_dev(x) -> torch.Tensor:
    t = to_dev(x)
    if t.dim() != 1:
        raise DimensionMismatch(f"expected 1-D vector, got shape {tuple(t.shape)}")
    return t


def mat_dev(x) -> torch.Tensor:
    t = to_dev(x)
    if t.dim() != 2:
        raise DimensionMismatch(f"expected 2-D matrix, got shape {tuple(t.shape)}")
    return t


def empty(n, *shape) -> torch.Tensor:
    return torch.empty((n, *shape), dtype=F64, device=device())


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def like_input(ref, t: torch.Tensor):
    """Return `t` as numpy if the caller passed host data, else as the device tensor."""
    return t if isinstance(ref, torch.Tensor) else to_host(t)
