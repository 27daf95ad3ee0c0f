"""Per-stream generators for the multi-PRNG tests: Philox4x32-10, SFC64, xoshiro256++.

The north star asks for these next to the reference's own Philox4x64-10 stream
(sampling.py): "SFC64/Xoshiro256++ are provided as per-stream kernels for the
multi-PRNG tests".  The reference's fixtures for them
(pkg/test_multi_prng_*.json) are orphaned -- nothing generates or reads them --
so these follow the published algorithms (see oracle/prng.c for the pins).
Kernels: csrc/prng.cu.  Device states live in int64 tensors holding the u64 bit
patterns; outputs are stream-major ``[n_streams, n]``.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import ConfigurationError

_U64 = (1 << 64) - 1


def _as_i64(words) -> np.ndarray:
    return np.asarray([int(w) & _U64 for w in np.ravel(words)], dtype=np.uint64).view(np.int64)


def philox4x32(key, counter, nblocks: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Philox4x32-10 words for counters counter .. counter+nblocks-1 (int32 bit patterns)."""
    k = [int(x) & 0xFFFFFFFF for x in key]
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in counter])
    out = torch.empty(4 * nblocks, dtype=torch.int32, device="cuda") if out is None else out
    _lib.call("simopt_philox4x32", _lib.stream_ptr(), k[0], k[1], c, nblocks, _lib.ptr(out))
    return out


class _Streams:
    _fn = ""

    def __init__(self, states: np.ndarray):
        st = np.ascontiguousarray(states, dtype=np.uint64).reshape(-1, 4)
        self.n_streams = st.shape[0]
        self.state = torch.from_numpy(st.view(np.int64).copy()).to("cuda")

    def _draw(self, n: int, kind: int) -> torch.Tensor:
        if n < 0:
            raise ConfigurationError("negative draw count")
        dt = torch.int64 if kind == 0 else torch.float64
        out = torch.empty(self.n_streams, n, dtype=dt, device="cuda")
        _lib.call(self._fn, _lib.stream_ptr(), _lib.ptr(self.state), self.n_streams, n, kind,
                  _lib.ptr(out))
        return out

    def raw(self, n: int) -> torch.Tensor:
        """[n_streams, n] 64-bit outputs (int64 bit patterns); advances every stream."""
        return self._draw(n, 0)

    def random(self, n: int) -> torch.Tensor:
        """[n_streams, n] doubles in [0, 1): (w >> 11) * 2^-53 (numpy's next_double)."""
        return self._draw(n, 1)

    def host_state(self) -> np.ndarray:
        return self.state.cpu().numpy().view(np.uint64)


class Sfc64Streams(_Streams):
    """SFC64 streams; state per stream = (a, b, c, counter) as numpy.random.SFC64."""

    _fn = "simopt_sfc64"

    @classmethod
    def from_seed(cls, seed: int, n_streams: int) -> "Sfc64Streams":
        """Stream k = numpy.random.SFC64(SeedSequence(seed).spawn(n_streams)[k])."""
        kids = np.random.SeedSequence(seed).spawn(n_streams)
        st = [np.random.SFC64(k).state["state"]["state"] for k in kids]
        return cls(np.array(st, dtype=np.uint64))


class Xoshiro256ppStreams(_Streams):
    """xoshiro256++ streams 2^128 steps apart (jump())."""

    _fn = "simopt_xoshiro256pp"

    @classmethod
    def from_state(cls, seed_state, n_streams: int) -> "Xoshiro256ppStreams":
        s = (ctypes.c_uint64 * 4)(*[int(x) & _U64 for x in seed_state])
        out = np.empty((n_streams, 4), dtype=np.uint64)
        lib = _lib.load(require_device=False)
        _lib.check(lib.simopt_xoshiro256pp_streams(s, n_streams, out.ctypes.data))
        return cls(out)
