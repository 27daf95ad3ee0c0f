"""Single-pass fused streaming evaluations (csrc/fused.cu, ABI simopt_fused_rows).

The reference evaluates every big pass as ``matvec`` then ``matvec_t`` over the
same matrix (mean-variance gradient tasks.py:78-85, logistic gradient
tasks.py:228-236, logistic HVP tasks.py:239-253): two reads of X.  The fused
kernel reads X once.  Its summation order is not the reference's fixed tree
(the exact-tree kernels stay the parity mode), so results agree to ~1e-15
relative -- inside the north star's 1e-10 gradient and 1e-8 trajectory gates.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ConfigurationError

MV, LR_GRAD, LR_HVP = 0, 1, 2


class SimoptPeerReduce(ctypes.Structure):
    """ctypes mirror of SimoptPeerReduce (include/simopt_b200.h)."""

    _fields_ = [("peers", ctypes.c_void_p), ("world", ctypes.c_int64), ("rank", ctypes.c_int64),
                ("seq", ctypes.c_uint64), ("status", ctypes.c_void_p)]


class PeerReducer:
    """Cross-rank sum fused into the fused passes' finish kernel over NVLink peer memory.

    One receive buffer per (shard, width) mapped into every rank with CUDA IPC
    (sharding.PeerMailbox); ``args()`` hands the kernel the next sequence number.
    ``get`` returns None on every rank when IPC is unavailable (callers then use
    raw partials + an NCCL allreduce).
    """

    _cache = {}

    def __init__(self, shard, mailbox, cols):
        self.shard, self.mailbox, self.cols = shard, mailbox, cols
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")

    @classmethod
    def get(cls, shard, cols: int):
        from .sharding import PeerMailbox
        key = (id(shard.group), shard.rank, shard.world, cols)
        if key not in cls._cache:
            nbytes = int(_lib.load().simopt_peer_reduce_bytes(shard.world, cols))
            mb = PeerMailbox.get(shard, nbytes=nbytes, tag=f"reduce{cols}")
            cls._cache[key] = None if mb is None else cls(shard, mb, cols)
        return cls._cache[key]

    def args(self) -> SimoptPeerReduce:
        a = SimoptPeerReduce()
        a.peers = self.mailbox.ptrs.data_ptr()
        a.world, a.rank = self.shard.world, self.shard.rank
        a.seq = self.mailbox.next_seq()
        a.status = self.status.data_ptr()
        return a

    def check(self):
        """Raise if any pass's exchange timed out (reads a device flag: synchronises)."""
        from .errors import DeviceError
        if int(self.status.item()):
            raise DeviceError("peer-memory allreduce timed out (a rank never arrived)")


def fused_geometry(mode: int, cols: int, vec: bool = True) -> dict:
    """The pass's launch geometry on this device: CTAs per cluster, resident clusters, grid."""
    c, n, g = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.call("simopt_fused_geometry", mode, cols, int(vec), ctypes.byref(c), ctypes.byref(n),
              ctypes.byref(g))
    return {"cluster": c.value, "clusters": n.value, "grid": g.value}


def fused_rows(mode: int, x: torch.Tensor, v: torch.Tensor, *, center=None, rowaux=None,
               col_scale: float = 1.0, col_out=None, scalar_out=None, t_out=None, dw_out=None,
               accumulate: bool = True, raw: bool = False, peer: PeerReducer | None = None):
    """One read of x (N x d, fp64, row-major, on the device); see include/simopt_b200.h.
    peer: sum the column sums and the scalar over the shard's ranks inside the pass."""
    n, d = x.shape
    if mode != MV and rowaux is None:  # (an empty row shard passes an empty weight tensor)
        raise ConfigurationError("row weights missing")
    P = _lib.ptr
    pa = None if peer is None else ctypes.byref(peer.args())
    _lib.call("simopt_fused_rows", _lib.stream_ptr(), int(mode), P(x), n, d, P(v), P(center),
              P(rowaux), float(col_scale), 1 if accumulate else 0, 1 if raw else 0, P(t_out), P(dw_out),
              P(col_out), P(scalar_out), pa)
    return col_out


def fused_rows_bits(mode: int, bits: torch.Tensor, d: int, v: torch.Tensor, *, rowaux,
                    col_scale: float = 1.0, col_out=None, scalar_out=None, t_out=None, dw_out=None,
                    accumulate: bool = True, raw: bool = False, peer: PeerReducer | None = None):
    """The logistic passes on bit-packed features (N x ceil(d/64) words)."""
    if rowaux is None:
        raise ConfigurationError("row weights missing")
    P = _lib.ptr
    pa = None if peer is None else ctypes.byref(peer.args())
    _lib.call("simopt_fused_rows_bits", _lib.stream_ptr(), int(mode), P(bits), bits.shape[0], d,
              P(v), P(rowaux), float(col_scale), 1 if accumulate else 0, 1 if raw else 0, P(t_out),
              P(dw_out), P(col_out), P(scalar_out), pa)
    return col_out
