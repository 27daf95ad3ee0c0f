"""Sample/product sharding across ranks (one process per GPU).

Reference anchor: the fixed tree of sobench/_kernels.py:1-42 (chunk partials
folded pairwise in index order).  If every rank owns whole 4096-chunks, the
allgathered per-chunk partials folded in index order reproduce the
single-process reduction bit for bit at any world size (SURVEY §8e
"deterministic mode").  RNG needs no communication: product j's draws are
normals j*S .. j*S+S-1 of the epoch's stream, i.e. Philox blocks
(j*S)//4 .. (j*S+S-1)//4.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

_U128 = (1 << 128) - 1


class SimoptComm:
    """The library's own NCCL communicator (simopt_comm_*, csrc/comm.cu).

    Rank 0 draws the 128-byte unique id, ``broadcast_id`` carries it to the other ranks
    (torch.distributed over the existing process group by default), every rank joins.
    Collectives run on the current CUDA stream, like every other entry point."""

    def __init__(self, rank: int, world: int, broadcast_id=None):
        import ctypes

        from . import _lib
        self.lib, self.rank, self.world = _lib.load(), rank, world
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            _lib.check(self.lib.simopt_comm_unique_id(ctypes.c_void_p(uid.data_ptr())))
        if world > 1:
            uid = (broadcast_id or _broadcast_id)(uid)
        self.handle = ctypes.c_void_p()
        _lib.check(self.lib.simopt_comm_init(ctypes.c_void_p(uid.data_ptr()), world, rank,
                                             ctypes.byref(self.handle)))

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        from . import _lib
        if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
            raise TypeError("simopt_comm_allreduce_f64 takes a contiguous float64 CUDA tensor")
        _lib.check(self.lib.simopt_comm_allreduce_f64(self.handle, _lib.stream_ptr(), _lib.ptr(t),
                                                      _lib.ptr(t), t.numel()))
        return t

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        from . import _lib
        t = t.contiguous()
        out = torch.empty((self.world, *t.shape), dtype=t.dtype, device=t.device)
        _lib.check(self.lib.simopt_comm_allgather(self.handle, _lib.stream_ptr(), _lib.ptr(t),
                                                  _lib.ptr(out), t.numel() * t.element_size()))
        return out

    def close(self):
        if self.handle:
            self.lib.simopt_comm_destroy(self.handle)
            self.handle = None


def _broadcast_id(uid: torch.Tensor) -> torch.Tensor:
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    t = uid.to(dev)
    dist.broadcast(t, 0)
    return t.cpu()


class ShardGroup:
    """The ranks that split one solver run's sample (or product) axis.

    Collectives go through ``torch.distributed``: NCCL over NVLink/NVSwitch on a
    GPU box (device tensors, issued on the current CUDA stream), or gloo (tensors
    staged through host memory -- the CPU tests and the two-processes-on-one-GPU
    parity tests).  Every rank runs the same program, so collectives are issued in
    the same order everywhere.
    """

    def __init__(self, group=None, comm: str | None = None):
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        # comm="simopt" (default with NCCL, env SIMOPT_COMM=torch to opt out): fp64 sums
        # and gathers of CUDA tensors go through the library's own NCCL communicator (the C
        # ABI a non-Python host uses); "torch": torch.distributed's
        import os
        comm = comm or os.environ.get("SIMOPT_COMM", "simopt")
        self.comm = None
        if self.nccl and self.world > 1 and group is None and comm == "simopt":
            self.comm = SimoptComm(self.rank, self.world)

    def range(self, n: int, align: int = 1) -> tuple:
        return shard_range(n, self.world, self.rank, align)

    def ranges(self, n: int, align: int = 1) -> list:
        return [shard_range(n, self.world, r, align) for r in range(self.world)]

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over ranks."""
        if self.world == 1:
            return t
        if self.comm is not None and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous():
            return self.comm.allreduce_(t)
        if self.nccl:
            dist.all_reduce(t, group=self.group)
            return t
        h = t.detach().cpu()
        dist.all_reduce(h, group=self.group)
        t.copy_(h)
        return t

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        """[world, *t.shape]: every rank's tensor, in rank order (equal shapes)."""
        t = t.contiguous()
        if self.world == 1:
            return t.unsqueeze(0)
        if self.comm is not None and t.is_cuda:
            return self.comm.allgather(t)
        if self.nccl:
            out = torch.empty((self.world, *t.shape), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t, group=self.group)
            return out
        h = t.detach().cpu()
        parts = [torch.empty_like(h) for _ in range(self.world)]
        dist.all_gather(parts, h, group=self.group)
        return torch.stack(parts).to(t.device)

    def allgather_rows(self, t: torch.Tensor, counts: list) -> torch.Tensor:
        """Concatenate each rank's first counts[r] rows (uneven shards, padded transfer)."""
        cap = max(max(counts), 1)
        pad = torch.zeros((cap, *t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        g = self.allgather(pad)
        return torch.cat([g[r, : counts[r]] for r in range(self.world)])

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)


def shifted_counter(counter: int, blocks: int) -> int:
    """Stream counter of a shard whose draws start `blocks` Philox blocks in (mod 2^128)."""
    return (counter + blocks) & _U128


def shard_range(n: int, world: int, rank: int, align: int = 4096) -> tuple:
    """[lo, hi) of rank's contiguous shard; boundaries are multiples of `align`."""
    units = -(-n // align)
    per = -(-units // world)
    lo = min(n, rank * per * align)
    hi = min(n, (rank + 1) * per * align)
    return lo, hi


def first_block(j: int, samples_per_item: int) -> tuple:
    """(Philox block index, word offset) of item j's first normal."""
    e = j * samples_per_item
    return e // 4, e % 4


def fold_pairwise(p: list) -> float:
    """_kernels.py:30-42 on a Python list (index order, odd tail carried)."""
    p = list(p)
    m = len(p)
    if m == 0:
        return 0.0
    while m > 1:
        h = m // 2
        q = [p[2 * i] + p[2 * i + 1] for i in range(h)]
        if m & 1:
            q.append(p[m - 1])
        p, m = q, len(q)
    return p[0]


def allgather_fold(local_partials: torch.Tensor, group=None) -> float:
    """Exact global tree root from each rank's in-order chunk partials (CPU or CUDA tensor)."""
    world = dist.get_world_size(group)
    n_local = torch.tensor([local_partials.numel()], dtype=torch.int64, device=local_partials.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    cap = int(max(s.item() for s in sizes))
    buf = torch.zeros(cap, dtype=torch.float64, device=local_partials.device)
    buf[: local_partials.numel()] = local_partials
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    parts = []
    for s, b in zip(sizes, bufs):
        parts.extend(b[: int(s.item())].cpu().tolist())
    return fold_pairwise(parts)


def allreduce_argmin(value: float, index: int, group=None, device="cpu") -> tuple:
    """Global first-argmin (np.argmin semantics) of per-rank (value, global index) pairs."""
    world = dist.get_world_size(group)
    t = torch.tensor([value, float(index)], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    best = None
    for o in out:
        v, i = float(o[0]), int(o[1])
        if best is None or v < best[0] or (v == best[0] and i < best[1]):
            best = (v, i)
    return best


class PeerMailbox:
    """Per-rank device mailbox mapped into every peer over CUDA IPC (NVLink/NVSwitch).

    Used by the newsvendor step kernel to exchange its LMO candidate with all ranks
    inside the kernel (csrc/newsvendor.cu nv_peer_exchange) instead of an NCCL
    allgather between launches.  Layout per rank: [2 parities][world][4 doubles].
    The sequence counter is monotonic for the mailbox's lifetime, so stale entries
    of earlier runs never match.  ``get`` returns None on every rank when any rank
    cannot map its peers (the caller then uses the NCCL exchange).
    """

    _cache = {}

    def __init__(self, shard: ShardGroup, nbytes: int | None = None):
        import ctypes

        from . import _lib
        lib = _lib.load()
        self.shard = shard
        W = shard.world
        self._own = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        nbytes = 2 * W * 4 * 8 if nbytes is None else nbytes
        _lib.check(lib.simopt_peer_alloc(nbytes, ctypes.byref(self._own), handle))
        handles = [None] * W
        dist.all_gather_object(handles, bytes(handle), group=shard.group)
        ptrs, self._opened = [], []
        for q in range(W):
            if q == shard.rank:
                ptrs.append(self._own.value)
                continue
            p = ctypes.c_void_p()
            _lib.check(lib.simopt_peer_open(handles[q], ctypes.byref(p)))
            self._opened.append(p)
            ptrs.append(p.value)
        self.ptrs = torch.tensor(ptrs, dtype=torch.int64, device="cuda")
        self.seq = 0
        # device-resident sequence for exchanges issued from replayed CUDA graphs
        self.seq_dev = torch.zeros(1, dtype=torch.int64, device="cuda")

    def next_seq(self) -> int:
        self.seq += 1
        return self.seq

    @classmethod
    def get(cls, shard: ShardGroup, nbytes: int | None = None, tag: str = "lmo"):
        """The (shard, tag) mailbox (default: the newsvendor LMO mailbox), created on first use."""
        key = (id(shard.group), shard.rank, shard.world, tag)
        if key in cls._cache:
            return cls._cache[key]
        try:
            mb, ok = cls(shard, nbytes), 1.0
        except Exception:  # noqa: BLE001 -- IPC unavailable here: every rank falls back
            mb, ok = None, 0.0
        flag = torch.tensor([ok], dtype=torch.float64, device="cuda" if shard.nccl else "cpu")
        if shard.world > 1:
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=shard.group)
        if float(flag.item()) < 1.0:
            mb = None
        cls._cache[key] = mb
        return mb
