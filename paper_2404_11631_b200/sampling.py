"""Counter-based random streams and samplers, generated on the B200.

Mirrors sobench/sampling.py (RngStream :51-80, uniform01 :87-102,
standard_normal :105-120, GaussianSpec :123-153, sample_returns :156-170,
sample_demands :173-193, sample_indices :196-209, synth_classification
:229-265).  A stream is (seed, stream_id, counter); block b of a draw is
Philox4x64-10 at counter + b + 1 with key (seed, stream_id) -- bit-identical to
numpy's Philox that the reference uses.  Normals use glibc-2.39-exact
Box-Muller on the device (csrc/glibc_math.cuh).

``*_device`` functions return CUDA tensors and never leave the GPU; the
reference-named functions return numpy arrays (drop-in, for parity tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import F64, device, empty, mat_dev, to_host, vec_dev
from .errors import (ConfigurationError, DimensionMismatch, EmptyRequest, InsufficientSamples,
                     InvalidConstraint)

_U64 = (1 << 64) - 1
_U128 = (1 << 128) - 1
_BLOCK = 4
SAMPLE_SPAN = 1 << 16  # sampling.py:46 (scheduling grid only; folded into the counter math)


@dataclass
class RngStream:
    """Reproducible random stream position; value-semantic and cheap to copy."""

    seed: int
    stream_id: int
    counter: int = 0

    def __post_init__(self):
        if not 0 <= self.seed <= _U64:
            raise ConfigurationError(f"seed must be a 64-bit unsigned int, got {self.seed}")
        if not 0 <= self.stream_id <= _U64:
            raise ConfigurationError(f"stream_id must be a 64-bit unsigned int, got {self.stream_id}")
        if not 0 <= self.counter <= _U128:
            raise ConfigurationError("counter must fit in 128 bits")

    def substream(self, stream_id: int) -> "RngStream":
        return RngStream(self.seed, stream_id)

    def clone(self) -> "RngStream":
        return RngStream(self.seed, self.stream_id, self.counter)

    # --- device addressing ---------------------------------------------------
    def words(self):
        """(seed, stream_id, ctr_lo, ctr_hi) as passed to the C ABI."""
        c = self.counter & _U128
        return self.seed, self.stream_id, c & _U64, (c >> 64) & _U64

    def advance(self, n_uniforms: int) -> None:
        self.counter += (n_uniforms + _BLOCK - 1) // _BLOCK


def uniform01_device(stream: RngStream, n: int, out: torch.Tensor | None = None) -> torch.Tensor:
    if n <= 0:
        raise EmptyRequest(f"requested {n} uniforms")
    out = empty(n) if out is None else out
    _lib.call("simopt_uniform01", _lib.stream_ptr(), *stream.words(), n, _lib.ptr(out))
    stream.advance(n)
    return out


def uniform01(stream: RngStream, n: int, backend=None) -> np.ndarray:
    """n doubles in [0, 1); advances the counter by ceil(n/4) blocks."""
    return to_host(uniform01_device(stream, n))


def standard_normal_device(stream: RngStream, n: int, out: torch.Tensor | None = None) -> torch.Tensor:
    if n <= 0:
        raise EmptyRequest(f"requested {n} normals")
    out = empty(n) if out is None else out
    _lib.call("simopt_standard_normal", _lib.stream_ptr(), *stream.words(), n, _lib.ptr(out))
    stream.advance(2 * ((n + 1) // 2))
    return out


def standard_normal(stream: RngStream, n: int, backend=None) -> np.ndarray:
    """n i.i.d. N(0,1) draws via Box-Muller on consecutive uniform pairs."""
    return to_host(standard_normal_device(stream, n))


@dataclass
class GaussianSpec:
    """Mean plus either a per-coordinate std or a lower-triangular factor (sampling.py:123-153)."""

    mean: object
    diag_std: object = None
    chol_factor: object = None

    def __post_init__(self):
        self.mean = np.ascontiguousarray(self.mean, dtype=np.float64)
        if self.mean.ndim != 1:
            raise DimensionMismatch("mean must be a vector")
        if (self.diag_std is None) == (self.chol_factor is None):
            raise ConfigurationError("provide exactly one of diag_std / chol_factor")
        if self.diag_std is not None:
            self.diag_std = np.ascontiguousarray(self.diag_std, dtype=np.float64)
            if self.diag_std.size != self.mean.size:
                raise DimensionMismatch("diag_std length != mean length")
            if not np.all(self.diag_std > 0):
                raise InvalidConstraint("diag_std entries must be > 0")
        else:
            self.chol_factor = np.ascontiguousarray(self.chol_factor, dtype=np.float64)
            d = self.mean.size
            if self.chol_factor.shape != (d, d):
                raise DimensionMismatch("chol_factor must be d x d")
            if not np.all(np.diag(self.chol_factor) > 0):
                raise InvalidConstraint("chol_factor diagonal must be > 0")
            if np.any(np.triu(self.chol_factor, 1) != 0):
                raise InvalidConstraint("chol_factor must be lower-triangular")

    @property
    def dimension(self) -> int:
        return self.mean.size


def sample_returns_device(spec: GaussianSpec, n_samples: int, stream: RngStream,
                          out: torch.Tensor | None = None, chunk: int = 4096) -> torch.Tensor:
    """N x d draws on the device; diag path fused (affine applied in-register)."""
    if n_samples < 2:
        raise InsufficientSamples(f"need at least 2 samples for a sample covariance, got {n_samples}")
    d = spec.dimension
    out = empty(n_samples, d) if out is None else out
    if spec.diag_std is not None:
        mu = vec_dev(spec.mean)
        sd = vec_dev(spec.diag_std)
        _lib.call("simopt_sample_returns_diag", _lib.stream_ptr(), *stream.words(), n_samples, d,
                  _lib.ptr(mu), _lib.ptr(sd), _lib.ptr(out))
        stream.advance(2 * ((n_samples * d + 1) // 2))
        return out
    # Cholesky path (sampling.py:167-170): out[i] = mean + fixed-tree matvec(L, z_i),
    # i.e. out[i, r] = tree-dot(L[r, :], z_i) -> one row-matvec of Z per factor row.
    z = standard_normal_device(stream, n_samples * d).view(n_samples, d)
    lt = mat_dev(spec.chol_factor)
    mu = vec_dev(spec.mean)
    col = empty(n_samples)
    for r in range(d):
        _lib.call("simopt_matvec", _lib.stream_ptr(), _lib.ptr(z), n_samples, d, None, n_samples,
                  None, _lib.ptr(lt[r]), chunk, _lib.ptr(col))
        out[:, r] = mu[r] + col
    return out


def sample_returns(spec: GaussianSpec, n_samples: int, stream: RngStream, backend=None) -> np.ndarray:
    chunk = getattr(backend, "chunk_size", 4096)
    return to_host(sample_returns_device(spec, n_samples, stream, chunk=chunk))


def sample_indices_device(n: int, b: int, stream: RngStream) -> torch.Tensor:
    """b indices from range(n), uniform without replacement (sampling.py:196-209).

    Partial Fisher-Yates with one uniform per selected index; the swap chain runs
    on the device (b <= 4096, the SQN mini-batches) or, for large b (instance
    label flips), in the native host helper over the device-drawn uniforms.
    """
    if not 1 <= b <= n:
        raise ConfigurationError(f"need 1 <= b <= n, got b={b}, n={n}")
    out = torch.empty(b, dtype=torch.int64, device=device())
    if b <= 4096:
        _lib.call("simopt_sample_indices", _lib.stream_ptr(), *stream.words(), n, b, _lib.ptr(out))
        stream.advance(b)
        return out
    u = uniform01(stream, b)
    host = np.empty(b, dtype=np.int64)
    _lib.check(_lib.load().simopt_fisher_yates_host(n, b, u.ctypes.data, host.ctypes.data))
    out.copy_(torch.from_numpy(host))
    return out


def sample_indices(n: int, b: int, stream: RngStream) -> np.ndarray:
    return to_host(sample_indices_device(n, b, stream))


class ClassificationData:
    """Synthetic binary-feature dataset on the device; labels carry the noise (sampling.py:212-226).

    Features are held either as fp64 0.0/1.0 (``features``, the reference's layout)
    or bit-packed (``bits``: u64 words, csrc/bits.cu layout -- 1/64 of the bytes;
    config 5's 10^7 x 8192 matrix is 10 GB instead of 655 GB).  Packed data
    materialises ``features`` on first access (device unpack) for the exact-tree
    paths; the fused Newton passes and the Hessian read the bits directly.
    """

    def __init__(self, features=None, labels=None, true_weights=None, shard=None, row_offset=0,
                 total_rows=None, bits=None, n_features=None):
        if features is None and bits is None:
            raise ConfigurationError("need features or bits")
        self._features = features
        self.bits = bits
        self.labels = labels            # this rank's rows, float64
        self.true_weights = true_weights
        self.shard = shard              # ShardGroup when the rows are split across ranks
        self.row_offset = row_offset    # first global row held here
        self.total_rows = total_rows
        self._d = features.shape[1] if features is not None else int(n_features)

    @property
    def features(self) -> torch.Tensor:
        if self._features is None:
            x = empty(max(self.local_rows, 0), self._d)
            _lib.call("simopt_unpack_bits", _lib.stream_ptr(), _lib.ptr(self.bits), self.local_rows,
                      self._d, _lib.ptr(x))
            self._features = x
        return self._features

    @property
    def packed(self) -> bool:
        return self.bits is not None

    def feature_major_u8(self):
        """(X^T as u8 in sample blocks, np): the integer-tensor-core Hessian's operand, built once."""
        if getattr(self, "_u8t", None) is None:
            if not self.packed:
                raise ConfigurationError("the u8 Hessian operand is built from bit-packed features")
            import ctypes
            n = self.local_rows
            ch, npv = ctypes.c_int64(), ctypes.c_int64()
            _lib.call("simopt_u8t_geometry", n, ctypes.byref(ch), ctypes.byref(npv))
            np_ = npv.value
            xt = torch.empty((np_ // ch.value) * self._d * (ch.value + 32), dtype=torch.uint8,
                             device=device())
            _lib.call("simopt_bits_to_u8t", _lib.stream_ptr(), _lib.ptr(self.bits), n, self._d, np_,
                      _lib.ptr(xt))
            self._u8t = (xt, np_)
        return self._u8t

    @property
    def n_samples(self) -> int:
        """Global row count N (the 1/N of every full-data average)."""
        return self.local_rows if self.total_rows is None else self.total_rows

    @property
    def local_rows(self) -> int:
        return (self._features if self._features is not None else self.bits).shape[0]

    @property
    def n_features(self) -> int:
        return self._d


def synth_classification(n_features: int, stream: RngStream, backend=None,
                         n_rows: int | None = None, shard=None, packed: bool = False) -> ClassificationData:
    """sampling.py:229-265, with the row count generalised (reference: n_rows = 30*n).

    X[i,j] = [u >= 0.5] is the MSB of the Philox word (written directly as 0.0/1.0);
    w_true continues the stream; scores use the fixed tree with chunk 4096 (the
    reference's module-level SequentialBackend); labels split at np.median; exactly
    floor(N/10) labels are flipped by sample_indices.
    """
    if n_features < 2:
        raise ConfigurationError(f"need at least 2 features, got {n_features}")
    n_rows = 30 * n_features if n_rows is None else int(n_rows)
    if shard is not None or packed:
        return _synth_classification_shard(n_features, stream, n_rows, shard, packed=packed)
    total = n_rows * n_features
    x = empty(n_rows, n_features)
    _lib.call("simopt_bernoulli_half", _lib.stream_ptr(), *stream.words(), total, _lib.ptr(x))
    stream.advance(total)
    w_true = standard_normal_device(stream, n_features)
    scores = empty(n_rows)
    _lib.call("simopt_matvec", _lib.stream_ptr(), _lib.ptr(x), n_rows, n_features, None, n_rows,
              None, _lib.ptr(w_true), 4096, _lib.ptr(scores))
    srt = torch.sort(scores).values  # order statistics for np.median (instance-time only)
    h = n_rows // 2
    if n_rows % 2:
        median = float(srt[h].item())
    else:
        a, b = float(srt[h - 1].item()), float(srt[h].item())
        median = (a + b) / 2.0  # np.median -> np.mean of the two middle values
    labels = empty(n_rows)
    _lib.call("simopt_threshold", _lib.stream_ptr(), _lib.ptr(scores), median, n_rows,
              _lib.ptr(labels))
    flip = sample_indices_device(n_rows, n_rows // 10, stream)
    labels[flip] = 1.0 - labels[flip]  # exact: labels are 0.0/1.0
    return ClassificationData(features=x, labels=labels, true_weights=w_true)


def _synth_classification_shard(n_features, stream, n_rows, shard, chunk=4096, packed=False):
    """Rows [lo, hi) of synth_classification (chunk-aligned; all rows without a shard),
    identical to the one-process instance: features are elements [lo*n, hi*n) of the
    same Philox draw, scores are row-local fixed-tree dots, the median is taken over
    the allgathered scores, and the replicated sample_indices flips are applied where
    they fall in [lo, hi).  packed: features generated straight into bits."""
    lo, hi = shard.range(n_rows, chunk) if shard is not None else (0, n_rows)
    nl = hi - lo
    total = n_rows * n_features
    if packed:
        W = -(-n_features // 64)
        bits = torch.empty(max(nl, 0), W, dtype=torch.int64, device=device())
        _lib.call("simopt_bernoulli_bits", _lib.stream_ptr(), *stream.words(), lo, hi, n_features,
                  _lib.ptr(bits))
        x = None
    else:
        x = empty(max(nl, 0), n_features)
        _lib.call("simopt_bernoulli_half_range", _lib.stream_ptr(), *stream.words(), lo * n_features,
                  hi * n_features, _lib.ptr(x))
    stream.advance(total)
    w_true = standard_normal_device(stream, n_features)
    scores = empty(max(nl, 1))
    if nl and packed:
        _lib.call("simopt_matvec_bits", _lib.stream_ptr(), _lib.ptr(bits), nl, n_features,
                  _lib.ptr(w_true), chunk, _lib.ptr(scores))
    elif nl:
        _lib.call("simopt_matvec", _lib.stream_ptr(), _lib.ptr(x), nl, n_features, None, nl,
                  None, _lib.ptr(w_true), chunk, _lib.ptr(scores))
    if shard is not None:
        counts = [b - a for a, b in shard.ranges(n_rows, chunk)]
        allsc = shard.allgather_rows(scores[:nl].view(-1, 1), counts).view(-1)
    else:
        allsc = scores[:nl]
    srt = torch.sort(allsc).values
    h = n_rows // 2
    if n_rows % 2:
        median = float(srt[h].item())
    else:
        median = (float(srt[h - 1].item()) + float(srt[h].item())) / 2.0
    labels = empty(max(nl, 1))
    if nl:
        _lib.call("simopt_threshold", _lib.stream_ptr(), _lib.ptr(scores), median, nl,
                  _lib.ptr(labels))
    flip = sample_indices_device(n_rows, n_rows // 10, stream)
    mine = flip[(flip >= lo) & (flip < hi)] - lo
    labels[mine] = 1.0 - labels[mine]
    return ClassificationData(features=x, labels=labels[:nl], true_weights=w_true, shard=shard,
                              row_offset=lo, total_rows=n_rows if shard is not None else None,
                              bits=bits if packed else None, n_features=n_features)
