"""The three problem definitions on the device (mirror of sobench/tasks.py).

Problem adapters implement the reference's duck-typed FW protocol
(``dimension/resample/gradient/lmo/check_feasible/objective``, frank_wolfe.py:91-121)
so the reference's own ``fw_run`` can drive them, and additionally
``fw_run_device``, the B200 path: the whole run is enqueued on one CUDA
stream and its trace is read back once per epoch.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import F64, empty, is_tensor, like_input, mat_dev, to_dev, to_host, vec_dev
from .errors import (ConfigurationError, DeviceError, DimensionMismatch, EmptyRequest, InsufficientSamples,
                     InvalidConstraint, InvalidGradient, RunAborted)
from .frank_wolfe import fw_step_size
from .fused import MV, fused_rows
from .lmo import SimplexSlackSet, lmo_general, lmo_simplex_slack, lmo_single_budget
from .records import TraceBuilder
from .sampling import GaussianSpec, RngStream

FEAS_TOL = 1e-10  # tasks.py:27


# ---------------------------------------------------------------------------
# ctypes mirror of NvIterArgs / NvState (include/simopt_b200.h)
class NvIterArgs(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int64), ("S", ctypes.c_int64), ("nseg", ctypes.c_int64),
        ("keys", ctypes.c_void_p), ("off", ctypes.c_void_p),
        ("seed", ctypes.c_uint64), ("sid", ctypes.c_uint64),
        ("ctr_lo", ctypes.c_uint64), ("ctr_hi", ctypes.c_uint64),
        ("mu", ctypes.c_void_p), ("sigma", ctypes.c_void_p), ("k", ctypes.c_void_p),
        ("h", ctypes.c_void_p), ("v", ctypes.c_void_p), ("c", ctypes.c_void_p),
        ("budget", ctypes.c_double),
        ("x_in", ctypes.c_void_p), ("x", ctypes.c_void_p), ("g", ctypes.c_void_p), ("terms", ctypes.c_void_p),
        ("gamma", ctypes.c_double),
        ("do_update", ctypes.c_int), ("do_grad", ctypes.c_int),
        ("step", ctypes.c_int64), ("grad_step", ctypes.c_int64),
        ("flags", ctypes.c_void_p), ("state", ctypes.c_void_p),
        ("part_v", ctypes.c_void_p), ("part_i", ctypes.c_void_p),
        ("part_capacity", ctypes.c_int64),
        ("peer_mb", ctypes.c_void_p), ("world", ctypes.c_int64), ("rank", ctypes.c_int64),
        ("j0", ctypes.c_int64), ("seq", ctypes.c_uint64),
        ("epoch_draw", ctypes.c_void_p), ("epoch_ctr", ctypes.c_void_p),
        ("inner_iters", ctypes.c_int64), ("m", ctypes.c_int64), ("seq_ptr", ctypes.c_void_p),
        ("stamp", ctypes.c_void_p),
    ]


def nv_geometry():
    """(draws per segment, buckets per segment) of the partitioned demand layout."""
    seg, nb = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("simopt_nv_geometry", ctypes.byref(seg), ctypes.byref(nb))
    return seg.value, nb.value


NV_FLAG_NAN_GRADIENT = 1
NV_FLAG_NEGATIVE = 2
NV_FLAG_EXCHANGE_TIMEOUT = 4
_NV_PART_CAPACITY = 16 * 148


# ---------------------------------------------------------------------------
# Task 2: multi-product newsvendor
@dataclass
class NewsvendorTask:
    """Per-product costs, Gaussian demand and the budget set (tasks.py:93-138).

    Either the single budget (``budget_costs``/``budget``, the benchmark default) or a
    multi-resource ``polytope`` (lmo.PolytopeSet, small instances: its FW steps run
    the generic loop with the device simplex LMO, csrc/lp.cu).
    """

    unit_cost: object
    holding_cost: object
    selling_value: object
    demand_mean: object
    demand_std: object
    budget_costs: object = None
    budget: float | None = None
    polytope: object = None

    def __post_init__(self):
        conv = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        self.unit_cost = conv(self.unit_cost)
        self.holding_cost = conv(self.holding_cost)
        self.selling_value = conv(self.selling_value)
        self.demand_mean = conv(self.demand_mean)
        self.demand_std = conv(self.demand_std)
        n = self.unit_cost.size
        for v in (self.holding_cost, self.selling_value, self.demand_mean, self.demand_std):
            if v.size != n:
                raise DimensionMismatch("newsvendor parameter vectors must share one length")
        if not np.all(self.selling_value + self.holding_cost > 0):
            raise InvalidConstraint("need v + h > 0 per product (convex per-product cost)")
        if not np.all(self.unit_cost - self.selling_value < 0):
            raise InvalidConstraint("need k - v < 0 per product (nondegenerate stocking)")
        if not np.all(self.demand_std > 0):
            raise InvalidConstraint("demand std must be > 0")
        has_budget = self.budget_costs is not None and self.budget is not None
        if has_budget == (self.polytope is not None):
            raise ConfigurationError("set exactly one of (budget_costs, budget) or polytope")
        if has_budget:
            self.budget_costs = conv(self.budget_costs)
            if self.budget_costs.size != n:
                raise DimensionMismatch("budget cost length mismatch")
            if not np.all(self.budget_costs > 0) or not self.budget > 0:
                raise InvalidConstraint("budget data must be strictly positive")
            self.budget = float(self.budget)

    @property
    def dimension(self) -> int:
        return self.unit_cost.size


class _NvDevice:
    """Device copies of a NewsvendorTask plus the epoch's keyed demand layout."""

    def __init__(self, task: NewsvendorTask, j0: int = 0, j1: int | None = None):
        # products [j0, j1) (the whole task unless product-sharded)
        j1 = task.dimension if j1 is None else j1
        self.j0, self.d_total = j0, task.dimension
        self.d = j1 - j0
        sl = slice(j0, j1)
        self.mu = to_dev(task.demand_mean[sl])
        self.sigma = to_dev(task.demand_std[sl])
        self.k = to_dev(task.unit_cost[sl])
        self.h = to_dev(task.holding_cost[sl])
        self.v = to_dev(task.selling_value[sl])
        self.c = to_dev(task.budget_costs[sl]) if task.budget_costs is not None else None
        self.budget = task.budget
        self.S = None
        self.keys = None
        self.off = None
        self.nseg = 0
        self.draw = None  # (seed, stream_id, ctr_lo, ctr_hi) of the epoch's draw
        # layout slots: the device FW loop double-buffers the epoch layout so the next
        # epoch's resample can run while this epoch's steps read the current one
        self.slots = {}   # slot -> [S, nseg, keys, off, draw]

    def ensure_layout(self, S: int, slot: int = 0, streams=()):
        """Layout slot for S draws per product.  `streams`: the side streams that read
        the slot's current buffers; a superseded buffer is kept from reuse until their
        queued work has run (the caching allocator only orders its own stream)."""
        cur = self.slots.get(slot)
        if cur is None or cur[0] != S:
            ns, ke, oe = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            _lib.call("simopt_nv_layout", self.d, S, ctypes.byref(ns), ctypes.byref(ke),
                      ctypes.byref(oe))
            if cur is not None:
                for st in streams:
                    cur[2].record_stream(st)
                    cur[3].record_stream(st)
            self.slots[slot] = None
            self.slots[slot] = [S, ns.value, torch.empty(ke.value, dtype=torch.int32, device="cuda"),
                                torch.empty(oe.value, dtype=torch.int16, device="cuda"), None]
        self.use_slot(slot)

    def use_slot(self, slot: int):
        self.S, self.nseg, self.keys, self.off, self.draw = self.slots[slot]

    def resample(self, stream: RngStream, S: int, slot: int = 0):
        if S < 1:
            raise InsufficientSamples("need at least one demand sample per product")
        self.ensure_layout(S, slot)
        # product j's draws are normals j*S .. j*S+S-1 of standard_normal(d*S): a shard
        # starting at product j0 (j0*S % 4 == 0) is the same draw with the counter
        # moved j0*S/4 Philox blocks on -- no RNG communication
        from .sharding import shifted_counter
        if self.j0:
            if (self.j0 * S) % 4:
                raise ConfigurationError("product shard must start on a Philox block")
            self.draw = RngStream(stream.seed, stream.stream_id,
                                  shifted_counter(stream.counter, self.j0 * S // 4)).words()
        else:
            self.draw = stream.words()
        self.slots[slot][4] = self.draw
        _lib.call("simopt_nv_resample", _lib.stream_ptr(), *self.draw, self.d, S,
                  _lib.ptr(self.keys), _lib.ptr(self.off))
        stream.advance(2 * ((self.d_total * S + 1) // 2))

    def counts(self, x: torch.Tensor) -> torch.Tensor:
        out = torch.empty(self.d, dtype=torch.int64, device="cuda")
        _lib.call("simopt_nv_counts", _lib.stream_ptr(), _lib.ptr(self.keys), _lib.ptr(self.off),
                  _lib.ptr(self.mu), _lib.ptr(self.sigma), self.d, self.S, *self.draw,
                  _lib.ptr(x), _lib.ptr(out))
        return out

    def decode(self) -> torch.Tensor:
        """Exact demand of every stored key (storage order) -- diagnostics/tests."""
        out = torch.empty(self.d * self.S, dtype=F64, device="cuda")
        _lib.call("simopt_nv_decode", _lib.stream_ptr(), _lib.ptr(self.keys), _lib.ptr(self.mu),
                  _lib.ptr(self.sigma), self.d, self.S, *self.draw, _lib.ptr(out))
        return out.view(self.d, self.S)


# fused mean-variance runs take the sample mean from simopt_col_sums_fast up to this many
# samples (above it the exact tree's column sums are HBM-bound anyway: C4 7.2 TB/s)
_FAST_MEAN_ROWS = 1 << 17


class NewsvendorProblem:
    """Newsvendor wired for FW: sampled gradient, exact recorded objective (tasks.py:293-334)."""

    name = "newsvendor"

    def __init__(self, task: NewsvendorTask, backend, shard=None, exchange: str = "peer"):
        self.task = task
        self.backend = backend
        # product sharding: products are independent; each FW step exchanges only the
        # per-rank LMO candidates -- "peer": inside the step kernel over NVLink peer
        # memory (sharding.PeerMailbox); "nccl": an allgather of 3 doubles per rank
        self.shard = shard
        if exchange not in ("peer", "nccl"):
            raise ConfigurationError(f"unknown exchange {exchange!r}")
        self.exchange = exchange
        if shard is not None and task.polytope is not None:
            raise ConfigurationError("product sharding needs the single-budget set (the "
                                     "multi-resource LMO couples all products)")
        j0, j1 = (0, task.dimension) if shard is None else shard.range(task.dimension, 4)
        if shard is not None and any(b <= a for a, b in shard.ranges(task.dimension, 4)):
            # every rank takes part in each step's LMO exchange with its own products
            raise ConfigurationError(
                f"product sharding of {task.dimension} products over {shard.world} ranks leaves "
                "a rank without products (shards are multiples of 4)")
        self.dev = _NvDevice(task, j0, j1)
        self._stream = None

    @property
    def dimension(self) -> int:
        return self.task.dimension

    # ---- duck-typed protocol (host arrays in/out, for the reference fw_run) ----
    def resample(self, stream: RngStream, n_samples: int) -> None:
        self.dev.resample(stream, n_samples)

    def _whole(self):
        if self.shard is not None:
            raise ConfigurationError("a product-sharded newsvendor runs through fw_run's device "
                                     "loop; per-call gradient/objective need the whole task")

    def gradient(self, x):
        self._whole()
        xd = vec_dev(x)
        cnt = self.dev.counts(xd)
        g = empty(self.dev.d)
        _lib.call("simopt_nv_grad_from_counts", _lib.stream_ptr(), _lib.ptr(cnt), self.dev.S,
                  _lib.ptr(self.dev.k), _lib.ptr(self.dev.h), _lib.ptr(self.dev.v), self.dev.d,
                  _lib.ptr(g))
        return like_input(x, g)

    def lmo(self, g):
        if self.task.polytope is not None:
            return lmo_general(g, self.task.polytope)
        return lmo_single_budget(g, self.dev.c if is_tensor(g) else self.task.budget_costs,
                                 self.task.budget)

    def project(self, y):
        """Euclidean projection onto {x >= 0, c.x <= C} (projected SGD, psgd.py)."""
        from .psgd import project_budget
        self._whole()
        return project_budget(y, self.dev.c, self.task.budget)

    def check_feasible(self, x) -> bool:
        self._whole()
        xd = vec_dev(x)
        if bool((xd < -FEAS_TOL).any()):
            return False
        if self.task.polytope is not None:  # tasks.py:330-332
            a, c = self.task.polytope.device()
            lhs = self.backend.matvec_device(a, xd)
            bound = empty(c.numel())
            _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(c), 1.0 + FEAS_TOL, None,
                      c.numel(), _lib.ptr(bound))
            return bool((lhs <= bound).all())
        spent = self.backend.dot(self.dev.c, xd)
        return float(spent) <= self.task.budget * (1.0 + FEAS_TOL)

    def objective(self, x) -> float:
        return nv_objective_exact(x, self.task, self.backend)

    # ---- B200 path ---------------------------------------------------------------
    def fw_run_device(self, config, backend, *, task_label, size, rep):
        """The fused device loop (single budget); None for a polytope task, whose steps
        take fw_run's generic loop (gradient, device simplex LMO, update, checks)."""
        if self.task.polytope is not None:
            return None
        return _nv_fw_run_device(self, config, backend, task_label, size, rep)


class NvFwEngine:
    """Device-resident Frank-Wolfe loop for one newsvendor run (frank_wolfe.py:91-121).

    Per step t (epoch k, inner m) the main stream runs ONE fused kernel: update x
    with the previous LMO vertex, compute the next ECDF gradient and its LMO argmin,
    and stamp %globaltimer when the step is done.  The recorded quantities of the
    epoch's M steps (exact-tree dot(c, x) for check_feasible, exact-tree objective
    sum) are formed by one launch on a side stream behind the epoch, off the critical
    path.  Iterates live in a ring of 2M+1 slots (an epoch's steps wait for the
    records of the epoch two back, the last reader of their slots), which also keeps
    the reference's final_iterate at hand when an epoch check finds a failure.
    """

    def __init__(self, prob: "NewsvendorProblem", inner_iters: int, epochs: int, chunk: int):
        dev = prob.dev
        self.prob, self.dev = prob, dev
        self.M, self.K, self.chunk = inner_iters, epochs, chunk
        d, M = dev.d, inner_iters
        T = epochs * M
        self.T, self.H = T, 2 * M + 1
        self.xs = torch.zeros(self.H, d, dtype=F64, device="cuda")
        self.g = empty(d)
        self.flags = torch.zeros(T + 1, dtype=torch.int32, device="cuda")
        self.spent = empty(T)
        self.objs = empty(T)
        self.stamps = torch.zeros(T + 1, dtype=torch.int64, device="cuda")
        self.state = torch.zeros(6, dtype=torch.int64, device="cuda")  # NvState (48 bytes)
        self.part_v = empty(_NV_PART_CAPACITY)
        self.part_i = torch.empty(_NV_PART_CAPACITY, dtype=torch.int64, device="cuda")
        a = NvIterArgs()
        a.d, a.mu, a.sigma = d, dev.mu.data_ptr(), dev.sigma.data_ptr()
        a.k, a.h, a.v, a.c = dev.k.data_ptr(), dev.h.data_ptr(), dev.v.data_ptr(), dev.c.data_ptr()
        a.budget = dev.budget
        a.g = self.g.data_ptr()
        a.flags, a.state = self.flags.data_ptr(), self.state.data_ptr()
        a.part_v, a.part_i, a.part_capacity = (self.part_v.data_ptr(), self.part_i.data_ptr(),
                                               _NV_PART_CAPACITY)
        self.args = a
        self.shard = prob.shard
        self.mailbox = None
        if self.shard is not None and prob.exchange == "peer":
            from .sharding import PeerMailbox
            self.mailbox = PeerMailbox.get(self.shard)  # None if IPC is unavailable (all ranks)
        if self.mailbox is not None:
            a.peer_mb = self.mailbox.ptrs.data_ptr()
            a.world, a.rank, a.j0 = self.shard.world, self.shard.rank, dev.j0
            a.seq_ptr = self.mailbox.seq_dev.data_ptr()  # one sequence source per mailbox
        if self.shard is not None:
            self.send = empty(3)
            # per epoch: spent[M] | objs[M] | nan[M+1] | negative[M+1] | timeout[M+1] flags
            self.red = empty(epochs, 5 * M + 3)
        self.lib = _lib.load()
        self.t0 = None
        self.resample_events = []
        # streams: FW steps (the critical path) at high priority; the next epoch's
        # resample (issue-bound, long) at low priority so step blocks are scheduled
        # first whenever resample blocks retire; recording sums on a side stream
        lo_pri, hi_pri = torch.cuda.Stream.priority_range() if hasattr(
            torch.cuda.Stream, "priority_range") else (0, -1)
        self.hi = torch.cuda.Stream(priority=hi_pri)
        self.gen = torch.cuda.Stream(priority=lo_pri)
        self.side = torch.cuda.Stream()
        self.epoch_done = {}  # epoch -> event after its last recorded step
        self.ready = {}       # epoch -> (layout slot, event: its resample is done)
        self.steps_done = {}  # epoch -> event after its last step kernel

    def start(self):
        cur = torch.cuda.current_stream()
        _lib.check(self.lib.simopt_timestamp(_lib.stream_ptr(cur), _lib.ptr(self.stamps[self.T:])))
        for s_ in (self.hi, self.gen, self.side):
            s_.wait_stream(cur)

    def _resample(self, k: int, stream: RngStream, n_samples: int, time_it: bool):
        """Epoch k's resample on the generator stream into layout slot k % 2."""
        slot = k % 2
        old = self.steps_done.get(k - 2)  # last reader of this slot
        if old is not None:
            self.gen.wait_event(old)
        # allocate on the caller's stream: the caching allocator keeps blocks per stream,
        # and a fresh engine's generator stream would otherwise cudaMalloc the layout anew
        self.dev.ensure_layout(n_samples, slot, streams=(self.hi, self.gen))
        with torch.cuda.stream(self.gen):
            if time_it:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            self.dev.resample(stream, n_samples, slot)
            if time_it:
                e1.record()
                self.resample_events.append((e0, e1))
            ev = torch.cuda.Event()
            ev.record()
        self.ready[k] = (slot, ev)

    def enqueue_epoch(self, k: int, stream: RngStream, n_samples: int, time_resample: bool = False,
                      next_samples: int | None = None):
        """Enqueue epoch k.  With next_samples, epoch k+1's resample is enqueued right
        behind this epoch's steps on the low-priority generator stream (it draws from
        `stream` after epoch k, exactly as a sequential run would) and overlaps them."""
        dev, a, lib, M, H = self.dev, self.args, self.lib, self.M, self.H
        if k not in self.ready:
            self._resample(k, stream, n_samples, time_resample)
        slot, ready = self.ready.pop(k)
        main = self.hi
        main.wait_event(ready)
        dev.use_slot(slot)
        sp = _lib.stream_ptr(main)
        ssp = _lib.stream_ptr(self.side)
        with torch.cuda.stream(main):
            self._enqueue_steps(k, sp, ssp)
        if next_samples is not None:
            self._resample(k + 1, stream, next_samples, time_resample)

    def _enqueue_steps(self, k: int, sp, ssp):
        dev, a, lib, M, H = self.dev, self.args, self.lib, self.M, self.H
        main = self.hi
        a.S, a.nseg = dev.S, dev.nseg
        a.keys, a.off = dev.keys.data_ptr(), dev.off.data_ptr()
        a.seed, a.sid, a.ctr_lo, a.ctr_hi = dev.draw
        t0 = k * M
        # ring slots (t0 + m + 1) % H were last written by epoch k-2's steps: its records
        # must have read them (H = 2M + 1)
        old = self.epoch_done.get(k - 2)
        if old is not None:
            main.wait_event(old)
        a.x_in = a.x = self.xs[t0 % H].data_ptr()  # gradient + LMO at the epoch's first iterate
        a.terms = None  # objective terms are formed with the epoch's records
        a.stamp = None
        a.do_update, a.do_grad, a.step, a.grad_step, a.gamma = 0, 1, t0, t0, 0.0
        self._seq()
        _lib.check(lib.simopt_nv_iter(sp, ctypes.byref(a)))
        self._exchange(sp)
        for m in range(M):
            t = t0 + m
            slot = (t + 1) % H
            xin, xout = self.xs[t % H], self.xs[slot]
            a.x_in, a.x = xin.data_ptr(), xout.data_ptr()
            a.gamma = fw_step_size(k, M, m)
            a.do_update, a.do_grad, a.step, a.grad_step = 1, int(m + 1 < M), t, t + 1
            a.stamp = self.stamps[t:].data_ptr()  # elapsed time of step t+1, on the device
            if m + 1 < M:
                self._seq()
            _lib.check(lib.simopt_nv_iter(sp, ctypes.byref(a)))
            if m + 1 < M:
                self._exchange(sp)
        a.stamp = None
        ev = torch.cuda.Event()
        ev.record(main)
        self.steps_done[k] = ev
        # the epoch's records in one launch, off the critical path: dot(c, x) for
        # check_feasible and the objective's vec_sum of newsvendor_cost_block, per step
        self.side.wait_event(ev)
        _lib.check(lib.simopt_nv_epoch_records(
            ssp, _lib.ptr(self.xs), H, (t0 + 1) % H, M, _lib.ptr(dev.c), _lib.ptr(dev.mu),
            _lib.ptr(dev.sigma), _lib.ptr(dev.k), _lib.ptr(dev.h), _lib.ptr(dev.v), dev.d, self.chunk,
            _lib.ptr(self.spent[t0:]), _lib.ptr(self.objs[t0:])))
        if self.shard is not None:
            self.epoch_done[k] = self._reduce_epoch(k)
        else:
            done = torch.cuda.Event()
            done.record(self.side)
            self.epoch_done[k] = done

    def _reduce_epoch(self, k: int):
        """Epoch totals over the product shards: one allreduce on the side stream, into a
        per-epoch row of self.red.  Returns the event after it."""
        M = self.M
        lo, hi = k * M, (k + 1) * M
        with torch.cuda.stream(self.side):
            r = self.red[k]
            r[:M].copy_(self.spent[lo:hi])
            r[M:2 * M].copy_(self.objs[lo:hi])
            f = self.flags[lo:hi + 1]
            r[2 * M:3 * M + 1].copy_((f & NV_FLAG_NAN_GRADIENT).to(F64))
            r[3 * M + 1:4 * M + 2].copy_((f & NV_FLAG_NEGATIVE).to(F64))
            r[4 * M + 2:].copy_((f & NV_FLAG_EXCHANGE_TIMEOUT).to(F64))
            self.shard.allreduce_(r)
            done = torch.cuda.Event()
            done.record(self.side)
        return done

    def _seq(self):
        """Next exchange sequence number (monotonic per mailbox, across runs)."""
        if self.mailbox is not None:
            self.args.seq = self.mailbox.next_seq()

    def _exchange(self, sp):
        """Global LMO vertex over product shards: allgather the per-rank argmins (NCCL
        path; the peer path exchanges inside the step kernel)."""
        if self.shard is None or self.mailbox is not None:
            return
        lib, P = self.lib, _lib.ptr
        _lib.check(lib.simopt_nv_lmo_pack(sp, P(self.state), self.dev.j0, P(self.send)))
        recv = self.shard.allgather(self.send)
        _lib.check(lib.simopt_nv_lmo_apply(sp, P(recv), self.shard.world, self.dev.j0, self.dev.d,
                                           P(self.state)))

    def finish(self):
        """Join the engine's streams into the caller's stream."""
        cur = torch.cuda.current_stream()
        for s_ in (self.hi, self.gen, self.side):
            cur.wait_stream(s_)

    def check_epoch(self, k: int, trace: TraceBuilder):
        """Append epoch k's rows to `trace`; return (t, exc, iterate) at the first failure."""
        M, H = self.M, self.H
        self.epoch_done[k].synchronize()
        lo, hi = k * M, (k + 1) * M
        if self.shard is None:
            fl = to_host(self.flags[lo:hi + 1])
            sp_ = to_host(self.spent[lo:hi])
            ob = to_host(self.objs[lo:hi])
        else:
            r = to_host(self.red[k])
            sp_, ob = r[:M], r[M:2 * M]
            fl = ((r[2 * M:3 * M + 1] > 0) * NV_FLAG_NAN_GRADIENT
                  + (r[3 * M + 1:4 * M + 2] > 0) * NV_FLAG_NEGATIVE
                  + (r[4 * M + 2:] > 0) * NV_FLAG_EXCHANGE_TIMEOUT).astype(np.int32)
        ts = to_host(self.stamps[lo:hi])
        if self.t0 is None:
            self.t0 = int(self.stamps[self.T].item())
        for i in range(M):
            t = lo + i
            if fl[i] & NV_FLAG_EXCHANGE_TIMEOUT:
                raise DeviceError(f"peer-memory LMO exchange timed out at step {t + 1}")
            if fl[i] & NV_FLAG_NAN_GRADIENT:
                return t, InvalidGradient("gradient contains NaN"), self.iterate(t, k)
            if (fl[i] & NV_FLAG_NEGATIVE) or not sp_[i] <= self.dev.budget * (1.0 + FEAS_TOL):
                return t, InvalidConstraint(f"iterate infeasible at step {t + 1}"), self.iterate(t + 1, k)
            trace.append(t + 1, float(ob[i]), int(ts[i]) - self.t0)
        return None

    def iterate(self, t: int, epoch: int | None = None) -> torch.Tensor:
        """Full iterate after step t (the product slices gathered when sharded); the
        ring of 2M+1 slots keeps it until two epochs later."""
        x = self.xs[t % self.H]
        if self.shard is None:
            return x
        counts = [b - a for a, b in self.shard.ranges(self.dev.d_total, 4)]
        return self.shard.allgather_rows(x.view(-1, 1), counts).view(-1)


class NvFwGraphEngine(NvFwEngine):
    """NvFwEngine whose epochs are replayed as CUDA graphs (one per epoch parity).

    Everything an epoch's step sequence reads is parity-fixed or device-resident, so
    the graph captured for parity p serves every epoch of that parity:
    * iterates live in two rings of M+1 rows; epoch k (parity p) starts from
      rings[1-p][M] (the previous epoch's last iterate) and writes rings[p][1..M];
    * the epoch's draw words and k sit in a per-parity device buffer (one pinned
      H2D copy per epoch); the step kernel reads them and forms
      gamma = 2 / (k M + m + 2) itself (frank_wolfe.py:62-66);
    * the peer LMO exchange's sequence number is a device counter;
    * flags and stamps go to per-parity buffers, copied into the per-epoch records
      right behind the replay; the epoch's recorded sums are one eager launch on the
      side stream behind the replay (simopt_nv_epoch_records), overlapping the next
      epoch.
    The host then enqueues one H2D copy and one graph launch per epoch instead of
    ~100 launches: the per-step host cost disappears, which is what bounds the
    product-sharded run at 8 GPUs (device time per step ~10 us).
    """

    def __init__(self, prob: "NewsvendorProblem", inner_iters: int, epochs: int, chunk: int):
        super().__init__(prob, inner_iters, epochs, chunk)
        d, M = self.dev.d, self.M
        self.rings = [torch.zeros(M + 1, d, dtype=F64, device="cuda") for _ in range(2)]
        self.flags_e = [torch.zeros(M + 1, dtype=torch.int32, device="cuda") for _ in range(2)]
        self.stamps_e = [torch.zeros(M, dtype=torch.int64, device="cuda") for _ in range(2)]
        self.host_params = [torch.zeros(5, dtype=torch.int64).pin_memory() for _ in range(2)]
        self.dev_params = [torch.zeros(5, dtype=torch.int64, device="cuda") for _ in range(2)]
        self.param_ev = [None, None]  # H2D of the parity's parameters (host buffer reuse)
        # the starting iterate of the last epoch of each parity (rings[1-p][M] is rewritten
        # by the next epoch of parity 1-p, which may already be queued when an epoch's
        # check needs it for RunAborted's final_iterate)
        self.starts = [torch.zeros(d, dtype=F64, device="cuda") for _ in range(2)]
        # graphs are keyed on everything a capture bakes in: parity and the layout slot's
        # (S, nseg, buffers) -- a sample schedule that changes S reallocates the slot
        self.graphs = {}
        self.warm = set()
        # captured kernel nodes keep the capture stream's priority: capture at high priority
        # so replayed steps still pre-empt the overlapping resample's blocks
        self.cstream = torch.cuda.Stream(priority=self.hi.priority)

    def _step_args(self, p: int, m: int, update: bool) -> NvIterArgs:
        """Arguments of step m (update + next gradient) or, m < 0, of the epoch's first gradient."""
        a = NvIterArgs.from_buffer_copy(self.args)
        dev, M = self.dev, self.M
        a.S, a.nseg = dev.slots[p][0], dev.slots[p][1]
        a.keys, a.off = dev.slots[p][2].data_ptr(), dev.slots[p][3].data_ptr()
        a.epoch_draw = self.dev_params[p].data_ptr()
        a.epoch_ctr = self.dev_params[p].data_ptr() + 4 * 8
        a.inner_iters, a.m = M, max(m, 0)
        a.flags = self.flags_e[p].data_ptr()
        a.terms = None
        prev_last = self.rings[1 - p][M].data_ptr()
        if not update:  # gradient + LMO at the epoch's first iterate
            a.x_in = a.x = prev_last
            a.do_update, a.do_grad, a.step, a.grad_step = 0, 1, 0, 0
        else:
            a.x_in = prev_last if m == 0 else self.rings[p][m].data_ptr()
            a.x = self.rings[p][m + 1].data_ptr()
            a.do_update, a.do_grad, a.step, a.grad_step = 1, int(m + 1 < M), m, m + 1
        return a

    def _steps(self, p: int, main):
        """The epoch's step sequence on `main`, capture-safe (the epoch's records are
        launched eagerly behind the replay, so they overlap the next epoch)."""
        lib, M = self.lib, self.M
        sp = _lib.stream_ptr(main)
        self.starts[p].copy_(self.rings[1 - p][M])
        _lib.check(lib.simopt_nv_iter(sp, ctypes.byref(self._step_args(p, -1, False))))
        for m in range(M):
            a = self._step_args(p, m, True)
            a.stamp = self.stamps_e[p][m:].data_ptr()
            _lib.check(lib.simopt_nv_iter(sp, ctypes.byref(a)))

    def enqueue_epoch(self, k: int, stream: RngStream, n_samples: int, time_resample: bool = False,
                      next_samples: int | None = None):
        if k not in self.ready:
            self._resample(k, stream, n_samples, time_resample)
        slot, ready = self.ready.pop(k)
        p = k & 1
        assert slot == p
        main = self.hi
        main.wait_event(ready)
        self.dev.use_slot(p)
        old = self.epoch_done.get(k - 2)  # its records read rings[p]
        if old is not None:
            main.wait_event(old)
        hp = self.host_params[p]
        if self.param_ev[p] is not None:  # the previous copy from this pinned buffer has run
            self.param_ev[p].synchronize()
        words = [w if w < (1 << 63) else w - (1 << 64) for w in self.dev.slots[p][4]]
        hp[:4] = torch.tensor(words, dtype=torch.int64)
        hp[4] = k
        with torch.cuda.stream(main):
            self.dev_params[p].copy_(hp, non_blocking=True)
            pe = torch.cuda.Event()
            pe.record(main)
            self.param_ev[p] = pe
            sl = self.dev.slots[p]
            key = (p, sl[0], sl[1], sl[2].data_ptr(), sl[3].data_ptr())
            g = self.graphs.get(key)
            if g is not None:
                g.replay()
            else:
                # first epoch of this layout: eager (allocations, library setup), then the
                # graph is captured right away, so a run's captures (a device sync each)
                # happen in its first two epochs -- inside any warm-up, never later
                self._steps(p, main)
                self.warm.add(key)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                self.cstream.wait_stream(main)
                with torch.cuda.graph(g, stream=self.cstream):
                    self._steps(p, self.cstream)
                self.graphs[key] = g
            steps = torch.cuda.Event()
            steps.record(main)
            # the parity buffers serve every epoch of that parity: copy this epoch's flags
            # and stamps out (on main, so epoch k+2's replay cannot overwrite them first)
            lo, hi, M = k * self.M, (k + 1) * self.M, self.M
            self.flags[lo:hi].copy_(self.flags_e[p][:M])
            self.flags_e[p].zero_()
            self.stamps[lo:hi].copy_(self.stamps_e[p])
            copied = torch.cuda.Event()
            copied.record(main)
        # the epoch's records (dot(c, x), objective) on the side stream, off the critical
        # path; rings[p] stays intact until epoch k+2, which waits for them
        dev, P = self.dev, _lib.ptr
        self.side.wait_event(steps)
        _lib.check(self.lib.simopt_nv_epoch_records(
            _lib.stream_ptr(self.side), P(self.rings[p]), M + 1, 1, M, P(dev.c), P(dev.mu), P(dev.sigma),
            P(dev.k), P(dev.h), P(dev.v), dev.d, self.chunk, P(self.spent[lo:]), P(self.objs[lo:])))
        self.side.wait_event(copied)
        done = torch.cuda.Event()
        done.record(self.side)
        self.steps_done[k] = steps
        self.epoch_done[k] = done
        if self.shard is not None:
            self.epoch_done[k] = self._reduce_epoch(k)
        if next_samples is not None:
            self._resample(k + 1, stream, next_samples, time_resample)

    def iterate(self, t: int, epoch: int | None = None) -> torch.Tensor:
        """Full iterate after t steps (product slices gathered when sharded), read as
        of `epoch` (default: the epoch whose steps produced it).  t = epoch*M is that
        epoch's start: its snapshot, which later epochs of the other parity cannot
        overwrite."""
        ke = max(t - 1, 0) // self.M if epoch is None else epoch
        m = t - ke * self.M
        x = self.starts[ke & 1] if m == 0 else self.rings[ke & 1][m]
        if self.shard is None:
            return x
        counts = [b - a for a, b in self.shard.ranges(self.dev.d_total, 4)]
        return self.shard.allgather_rows(x.view(-1, 1), counts).view(-1)


def make_nv_engine(prob: "NewsvendorProblem", inner_iters: int, epochs: int, chunk: int,
                   graph: bool | None = None):
    """Engine for a device FW run.  graph=None: CUDA-graph epochs for product-sharded runs
    with the peer-memory exchange (per-step device work ~10 us at 8 GPUs, so host launch
    cost would bound them); the eager engine otherwise (on one GPU the epoch is device-bound
    and eager launching measured as fast; NCCL exchanges are not captured)."""
    eng = NvFwEngine(prob, inner_iters, epochs, chunk)
    if graph is None:
        graph = eng.mailbox is not None
    if not graph or (prob.shard is not None and eng.mailbox is None):
        return eng
    return NvFwGraphEngine(prob, inner_iters, epochs, chunk)


def _nv_fw_run_device(prob: "NewsvendorProblem", config, backend, label, size, rep):
    eng = make_nv_engine(prob, config.inner_iters, config.epochs, backend.chunk_size)
    trace = TraceBuilder()

    def abort(t, exc, it):
        partial = trace.build(label, size, backend.kind, rep, config.stream.seed, to_host(it))
        raise RunAborted(f"frank-wolfe run failed at step {len(trace) + 1}: {exc}", partial) from exc

    eng.start()
    for k in range(config.epochs):
        nxt = config.epoch_sample_size(k + 1) if k + 1 < config.epochs else None
        eng.enqueue_epoch(k, config.stream, config.epoch_sample_size(k), next_samples=nxt)
        if k >= 1:  # validate the previous epoch (waits for its records) while this one runs
            bad = eng.check_epoch(k - 1, trace)
            if bad:
                abort(*bad)
    eng.finish()
    bad = eng.check_epoch(config.epochs - 1, trace)
    if bad:
        abort(*bad)
    return trace.build(label, size, backend.kind, rep, config.stream.seed, to_host(eng.iterate(eng.T)))


def sample_demands_device(mu, sigma, n_samples: int, stream: RngStream) -> torch.Tensor:
    """sample_demands (sampling.py:173-193) on the device: per-product demand draws, each
    row sorted ascending, bit-identical to the reference's matrix.

    The draw is the FW loop's own keyed resample (k_nv_resample, the same Philox/glibc
    normals z[j*S + s]); k_nv_decode evaluates every draw's exact demand mu_j + sigma_j*z
    (sampling.py:191) and the rows are sorted by value (no arithmetic).  The FW loop
    itself never materialises this matrix -- it is the reference-format view of an
    epoch for callers of the reference API."""
    mud, sgd = vec_dev(mu), vec_dev(sigma)
    if mud.numel() != sgd.numel():
        raise DimensionMismatch("mu and sigma lengths differ")
    if not bool((sgd > 0).all()):
        raise InvalidConstraint("sigma entries must be > 0")
    if n_samples < 1:
        raise EmptyRequest("need at least one demand sample per product")
    d, S = mud.numel(), int(n_samples)
    ns, ke, oe = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.call("simopt_nv_layout", d, S, ctypes.byref(ns), ctypes.byref(ke), ctypes.byref(oe))
    keys = torch.empty(ke.value, dtype=torch.int32, device="cuda")
    off = torch.empty(oe.value, dtype=torch.int16, device="cuda")
    draw = stream.words()
    _lib.call("simopt_nv_resample", _lib.stream_ptr(), *draw, d, S, _lib.ptr(keys), _lib.ptr(off))
    stream.advance(2 * ((d * S + 1) // 2))
    out = torch.empty(d, S, dtype=F64, device="cuda")
    _lib.call("simopt_nv_decode", _lib.stream_ptr(), _lib.ptr(keys), _lib.ptr(mud), _lib.ptr(sgd),
              d, S, *draw, _lib.ptr(out))
    return torch.sort(out, dim=1).values


def sample_demands(mu, sigma, n_samples: int, stream: RngStream, backend=None) -> np.ndarray:
    return to_host(sample_demands_device(mu, sigma, n_samples, stream))


def nv_gradient_hat(x, demands, task: NewsvendorTask, backend):
    """k - v + (h+v) * empirical CDF at x (tasks.py:141-160) on reference-format sorted rows."""
    dem = mat_dev(demands)
    xd = vec_dev(x)
    if dem.shape[0] != xd.numel():
        raise DimensionMismatch("demand rows != product count")
    if dem.shape[1] == 0:
        raise InsufficientSamples("empty demand sample array")
    cnt = torch.empty(xd.numel(), dtype=torch.int64, device="cuda")
    _lib.call("simopt_ecdf_count_sorted", _lib.stream_ptr(), _lib.ptr(dem), dem.shape[0],
              dem.shape[1], _lib.ptr(xd), _lib.ptr(cnt))
    k, h, v = (to_dev(a) for a in (task.unit_cost, task.holding_cost, task.selling_value))
    g = empty(xd.numel())
    _lib.call("simopt_nv_grad_from_counts", _lib.stream_ptr(), _lib.ptr(cnt), dem.shape[1],
              _lib.ptr(k), _lib.ptr(h), _lib.ptr(v), xd.numel(), _lib.ptr(g))
    return like_input(x, g)


def nv_gradient_exact(x, task: NewsvendorTask, backend):
    """k - v + (h+v) * Phi((x - mu)/sigma), the exact Gaussian CDF (tasks.py:163-171)."""
    xd = vec_dev(x)
    if xd.numel() != task.dimension:
        raise DimensionMismatch("stock vector length != product count")
    dev = [to_dev(a) for a in (task.demand_mean, task.demand_std, task.unit_cost,
                               task.holding_cost, task.selling_value)]
    g = empty(xd.numel())
    _lib.call("simopt_nv_grad_exact", _lib.stream_ptr(), _lib.ptr(xd), *(_lib.ptr(t) for t in dev),
              xd.numel(), _lib.ptr(g))
    return like_input(x, g)


def nv_objective_exact(x, task: NewsvendorTask, backend) -> float:
    """Expected cost under Gaussian demand, fixed-tree sum (tasks.py:174-188)."""
    xd = vec_dev(x)
    if xd.numel() != task.dimension:
        raise DimensionMismatch("stock vector length != product count")
    terms = nv_cost_terms_device(xd, task)
    return backend.vec_sum(terms) if is_tensor(x) else float(backend.vec_sum_device(terms).item())


def nv_cost_terms_device(xd, task: NewsvendorTask):
    out = empty(xd.numel())
    dev = [to_dev(a) for a in (task.demand_mean, task.demand_std, task.unit_cost,
                               task.holding_cost, task.selling_value)]
    _lib.call("simopt_nv_cost_terms", _lib.stream_ptr(), _lib.ptr(xd), *(_lib.ptr(t) for t in dev),
              xd.numel(), _lib.ptr(out))
    return out


# ---------------------------------------------------------------------------
# Task 1: mean-variance portfolio
@dataclass
class MeanVarTask:
    """Return distribution for the mean-variance objective (tasks.py:33-41)."""

    spec: GaussianSpec

    @property
    def dimension(self) -> int:
        return self.spec.dimension


class MeanVarSampleSet:
    """One epoch's draws X (N x d, device), their column mean, and N (tasks.py:44-53).

    The centered matrix Xc = X - mean is never stored: every kernel subtracts
    the mean on the fly, which is the same IEEE subtraction numpy performs
    when materialising it (tasks.py:63).  ``centered`` materialises on demand.
    """

    def __init__(self, samples: torch.Tensor, mean: torch.Tensor, count: int | None = None):
        self.samples = samples  # this rank's rows when sharded
        self.mean = mean
        self.count = samples.shape[0] if count is None else count  # global N

    @property
    def centered(self) -> torch.Tensor:
        return self.samples - self.mean[None, :]


def build_sample_set(samples, backend, mean_out=None) -> MeanVarSampleSet:
    """colsum = tree matvec_t(X, 1); mean = colsum * (1/n) (tasks.py:56-64)."""
    x = mat_dev(samples)
    n = x.shape[0]
    if n < 2:
        raise InsufficientSamples("sample covariance needs at least 2 rows")
    ones = torch.ones(n, dtype=F64, device="cuda")
    col = backend.matvec_t_device(x, ones)
    mean = empty(x.shape[1]) if mean_out is None else mean_out
    _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(col), 1.0 / n, None, col.numel(),
              _lib.ptr(mean))
    return MeanVarSampleSet(x, mean)


def mv_objective(w, ss: MeanVarSampleSet, backend) -> float:
    """0.5/(N-1) * |Xc w|^2 - w.mean (tasks.py:67-75)."""
    wd = vec_dev(w)
    if wd.numel() != ss.mean.numel():
        raise DimensionMismatch("weight length != asset count")
    q = backend.matvec_device(ss.samples, wd, center=ss.mean)
    quad = float(backend.dot_device(q, q).item())
    lin = float(backend.dot_device(wd, ss.mean).item())
    return 0.5 * quad / (ss.count - 1) - lin


def mv_gradient(w, ss: MeanVarSampleSet, backend):
    """(1/(N-1)) Xc^T (Xc w) - mean (tasks.py:78-85)."""
    wd = vec_dev(w)
    if wd.numel() != ss.mean.numel():
        raise DimensionMismatch("weight length != asset count")
    q = backend.matvec_device(ss.samples, wd, center=ss.mean)
    gq = backend.matvec_t_device(ss.samples, q, center=ss.mean)
    g = empty(gq.numel())
    _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(gq), 1.0 / (ss.count - 1),
              _lib.ptr(ss.mean), gq.numel(), _lib.ptr(g))
    return like_input(w, g)


# --- deterministic sample sharding -------------------------------
# A rank owns rows [lo, hi) with lo, hi on chunk boundaries, so its matvec_t chunk
# partials ARE the reference's partials of those chunks; gathered in rank order and
# folded they give the single-process fixed-tree result bit for bit at any world size.
def _chunk_counts(shard, n, chunk):
    return [-(-(hi - lo) // chunk) for lo, hi in shard.ranges(n, chunk)]


def sharded_matvec_t(shard, a_loc, x_loc, n_total, chunk, center=None, out=None):
    """Fixed-tree a^T x over row shards (backend.py:128-141 across ranks)."""
    cols = a_loc.shape[1]
    nloc = -(-a_loc.shape[0] // chunk)
    part = empty(max(nloc, 1), cols)
    if nloc:
        _lib.call("simopt_matvec_t_partials", _lib.stream_ptr(), _lib.ptr(a_loc), a_loc.shape[0],
                  cols, _lib.ptr(center), _lib.ptr(x_loc), chunk, _lib.ptr(part))
    counts = _chunk_counts(shard, n_total, chunk)
    allp = shard.allgather_rows(part[:nloc], counts)
    out = empty(cols) if out is None else out
    _lib.call("simopt_fold_partials", _lib.stream_ptr(), _lib.ptr(allp), allp.shape[0], cols,
              _lib.ptr(out))
    return out


def sharded_dot(shard, x_loc, y_loc, n_total, chunk, out=None):
    """Fixed-tree dot over row shards (dot partials = matvec_t of the n x 1 matrix)."""
    return sharded_matvec_t(shard, x_loc.view(-1, 1), y_loc, n_total, chunk, out=out)


class MeanVarProblem:
    """Mean-variance task wired for the FW engine (tasks.py:261-290)."""

    name = "meanvar"

    def __init__(self, task: MeanVarTask, backend, fused: bool = False, shard=None,
                 exchange: str = "peer"):
        self.task = task
        self.backend = backend
        self.fused = fused  # device FW loop: single-pass fused gradient (csrc/fused.cu)
        # sample sharding: this rank draws and reduces only its scenario rows
        # [lo, hi) (chunk-aligned), with one allreduce / allgather per reduction; fused
        # mode sums across ranks inside the pass's finish kernel over peer memory
        # ("peer"; NCCL allreduce of raw partials if unavailable, or with "nccl")
        self.shard = shard
        if exchange not in ("peer", "nccl"):
            raise ConfigurationError(f"unknown exchange {exchange!r}")
        self.exchange = exchange
        self.constraint = SimplexSlackSet(task.dimension)
        self.sample_set: MeanVarSampleSet | None = None
        self._x = None
        self._mean = empty(task.dimension)
        self._engines = {}

    @property
    def dimension(self) -> int:
        return self.task.dimension

    def resample(self, stream: RngStream, n_samples: int) -> None:
        from .sampling import sample_returns_device
        d = self.dimension
        if self.shard is not None:
            self._resample_shard(stream, n_samples)
            return
        if self._x is None or self._x.shape[0] != n_samples:
            self._x = None
            self._x = empty(n_samples, d)
        x = sample_returns_device(self.task.spec, n_samples, stream, out=self._x,
                                  chunk=self.backend.chunk_size)
        self.sample_set = build_sample_set(x, self.backend, mean_out=self._mean)

    def resample_slot(self, stream: RngStream, n_samples: int, slot: int) -> MeanVarSampleSet:
        """Epoch draw into buffer `slot` (0/1) on the current stream: the device FW loop
        double-buffers X so the next epoch's draw overlaps this epoch's steps.  Diagonal
        model, unsharded; the same draws and exact-tree mean as resample()."""
        spec, d = self.task.spec, self.dimension
        if n_samples < 2:
            raise InsufficientSamples(f"need at least 2 samples for a sample covariance, got {n_samples}")
        if not hasattr(self, "_slots"):
            self._slots = {}
            self._mu_dev, self._sd_dev = vec_dev(spec.mean), vec_dev(spec.diag_std)
        cur = self._slots.get(slot)
        if cur is None or cur[0].shape[0] != n_samples:
            self._slots[slot] = None
            self._slots[slot] = (empty(n_samples, d), empty(d),
                                 torch.ones(n_samples, dtype=F64, device="cuda"))
        x, mean, ones = self._slots[slot]
        _lib.call("simopt_sample_returns_diag", _lib.stream_ptr(), *stream.words(), n_samples, d,
                  _lib.ptr(self._mu_dev), _lib.ptr(self._sd_dev), _lib.ptr(x))
        stream.advance(2 * ((n_samples * d + 1) // 2))
        if self.fused and n_samples <= _FAST_MEAN_ROWS:
            # fused mode (trajectories within 1e-8, not the tree): the column sums in a fixed
            # order of 256 short chains -- at C1's N the tree's 4096-long chains are latency-
            # bound (81 vs ~10 us) and trail the next epoch's draw
            col = empty(d)
            _lib.call("simopt_col_sums_fast", _lib.stream_ptr(), _lib.ptr(x), n_samples, d, _lib.ptr(col))
        else:
            col = self.backend.matvec_t_device(x, ones)      # build_sample_set (tasks.py:56-64)
        _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(col), 1.0 / n_samples, None, d,
                  _lib.ptr(mean))
        return MeanVarSampleSet(x, mean)

    def _resample_shard(self, stream: RngStream, n_samples: int) -> None:
        """Rows [lo, hi) of sample_returns (no RNG communication) + the exact global mean."""
        spec, d, chunk = self.task.spec, self.dimension, self.backend.chunk_size
        if n_samples < 2:
            raise InsufficientSamples(f"need at least 2 samples for a sample covariance, got {n_samples}")
        if spec.diag_std is None:
            raise ConfigurationError("sample sharding supports the diagonal return model")
        lo, hi = self.shard.range(n_samples, chunk)
        if self._x is None or self._x.shape[0] != hi - lo:
            self._x = None
            self._x = empty(max(hi - lo, 0), d)
        mu, sd = vec_dev(spec.mean), vec_dev(spec.diag_std)
        _lib.call("simopt_sample_returns_diag_rows", _lib.stream_ptr(), *stream.words(), lo, hi, d,
                  _lib.ptr(mu), _lib.ptr(sd), _lib.ptr(self._x))
        stream.advance(2 * ((n_samples * d + 1) // 2))
        ones = torch.ones(max(hi - lo, 1), dtype=F64, device="cuda")
        col = sharded_matvec_t(self.shard, self._x, ones, n_samples, chunk)
        _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(col), 1.0 / n_samples, None, d,
                  _lib.ptr(self._mean))
        self.sample_set = MeanVarSampleSet(self._x, self._mean, count=n_samples)

    def objective(self, w) -> float:
        if self.shard is None and self.fused:
            ss, wd = self.sample_set, vec_dev(w)
            quad = empty(1)
            fused_rows(MV, ss.samples, wd, center=ss.mean, scalar_out=quad, accumulate=False)
            lin = float(self.backend.dot_device(wd, ss.mean).item())
            return 0.5 * float(quad.item()) / (ss.count - 1) - lin
        if self.shard is None:
            return mv_objective(w, self.sample_set, self.backend)
        ss, chunk, wd = self.sample_set, self.backend.chunk_size, vec_dev(w)
        q = self.backend.matvec_device(ss.samples, wd, center=ss.mean)
        quad = float(sharded_dot(self.shard, q, q, ss.count, chunk).item())
        lin = float(self.backend.dot_device(wd, ss.mean).item())
        return 0.5 * quad / (ss.count - 1) - lin

    def gradient(self, w):
        if self.shard is None and self.fused:  # one read of X (csrc/fused.cu)
            ss, wd = self.sample_set, vec_dev(w)
            g = empty(wd.numel())
            fused_rows(MV, ss.samples, wd, center=ss.mean, col_scale=1.0 / (ss.count - 1), col_out=g)
            return like_input(w, g)
        if self.shard is None:
            return mv_gradient(w, self.sample_set, self.backend)
        ss, chunk, wd = self.sample_set, self.backend.chunk_size, vec_dev(w)
        q = self.backend.matvec_device(ss.samples, wd, center=ss.mean)
        gq = sharded_matvec_t(self.shard, ss.samples, q, ss.count, chunk, center=ss.mean)
        g = empty(gq.numel())
        _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(gq), 1.0 / (ss.count - 1),
                  _lib.ptr(ss.mean), gq.numel(), _lib.ptr(g))
        return like_input(w, g)

    def lmo(self, g):
        return lmo_simplex_slack(g)

    def project(self, y):
        """Euclidean projection onto {w >= 0, sum(w) <= 1} (projected SGD, psgd.py)."""
        from .psgd import project_budget
        return project_budget(y, None, 1.0)

    def check_feasible(self, w) -> bool:
        wh = to_host(w) if is_tensor(w) else np.asarray(w)
        return bool(np.all(wh >= -FEAS_TOL) and np.sum(wh) <= 1.0 + FEAS_TOL)

    def fw_run_device(self, config, backend, *, task_label, size, rep):
        return _mv_fw_run_device(self, config, backend, task_label, size, rep)


class MvFwEngine:
    """Device-resident Frank-Wolfe loop for the mean-variance task (frank_wolfe.py:91-121).

    The M inner steps of an epoch are captured as a CUDA graph (one per iterate
    ring, two rings alternating by epoch parity) and replayed every epoch: at C1
    sizes a step is ~8 latency-bound kernels, so launch overhead would otherwise
    dominate.  Everything that changes between epochs lives in device memory the
    graph reads: the iterate ring (slot 0 = the epoch's first iterate), the step
    sizes gamma (copied in before each replay) and the epoch-local trace buffers
    (copied out after).  q = Xc w_{t+1} of the objective is reused as the first
    half of gradient(w_{t+1}) inside an epoch (same kernel, same bits).
    Feasibility: min(w) and an exact-tree sum (the reference uses numpy's
    pairwise np.sum, tasks.py:290; both are within 1e-15 of the exact sum, far
    inside the 1e-10 tolerance of that boolean test).

    ``fused``: each step is ONE read of X -- the single-pass kernel evaluated at
    w_{t+1} yields |Xc w_{t+1}|^2 for objective(t) and the full gradient at
    w_{t+1} for step t+1 (the last step of an epoch skips the unused column
    sums): M+1 passes per epoch instead of 2M+1, in a fast summation order
    (trajectories within 1e-8 of the exact tree).
    """

    def __init__(self, prob: "MeanVarProblem", inner_iters: int, chunk: int, use_graph: bool = True):
        self.prob, self.M, self.chunk, self.use_graph = prob, inner_iters, chunk, use_graph
        d, M = prob.dimension, inner_iters
        self.rings = [torch.zeros(M + 1, d, dtype=F64, device="cuda") for _ in range(2)]
        self.g, self.gq, self.s, self.dirn = empty(d), empty(d), empty(d), empty(d)
        self.gamma = empty(M)
        # per-parity pinned staging of the epoch's step sizes: a pageable host-to-device copy
        # synchronises the stream, i.e. would hold the host until the previous epoch ends
        self._gamma_pin = [torch.empty(M, dtype=F64, pin_memory=True) for _ in range(2)]
        self.status = torch.zeros(M, dtype=torch.int32, device="cuda")
        self.wmin, self.wsum, self.quad, self.lin = empty(M), empty(M), empty(M), empty(M)
        self.stamps = torch.zeros(M, dtype=torch.int64, device="cuda")
        self.q = None
        self.red_buf = empty(d + 1)
        self.graphs = {}
        self.warm = False
        self.cstream = torch.cuda.Stream()  # capture stream: its library scratch is pre-warmed
        self.lib = _lib.load()

    def _steps(self, ws, x, mean, n_k):
        """Enqueue the M inner steps on the current stream (captured or eager)."""
        lib, sp, chunk, d, q = self.lib, _lib.stream_ptr(), self.chunk, self.prob.dimension, self.q
        inv = 1.0 / (n_k - 1)
        P = _lib.ptr
        if self.prob.shard is not None:
            self._sharded_steps(ws, x, mean, n_k, inv)
            return
        if self.prob.fused:
            self._fused_steps(ws, x, mean, n_k, inv)
            return
        for m in range(self.M):
            w_in, w_out = ws[m], ws[m + 1]
            if m == 0:  # first gradient of the epoch: q = Xc w_kM
                _lib.check(lib.simopt_matvec(sp, P(x), n_k, d, None, n_k, P(mean), P(w_in), chunk, P(q)))
            _lib.check(lib.simopt_matvec_t(sp, P(x), n_k, d, None, n_k, P(mean), P(q), chunk, P(self.gq)))
            _lib.check(lib.simopt_scale_sub(sp, P(self.gq), inv, P(mean), d, P(self.g)))
            self._tail(sp, m, w_in, w_out, mean)
            # objective(w_{t+1}); q is reused by the next gradient of this epoch
            _lib.check(lib.simopt_matvec(sp, P(x), n_k, d, None, n_k, P(mean), P(w_out), chunk, P(q)))
            _lib.check(lib.simopt_dot(sp, P(q), P(q), n_k, chunk, P(self.quad[m:])))
            _lib.check(lib.simopt_timestamp(sp, P(self.stamps[m:])))

    def _tail(self, sp, m, w_in, w_out, mean):
        """LMO + update + min + exact sum/dot of the new iterate: one launch (simopt_mv_fw_tail)."""
        P = _lib.ptr
        _lib.check(self.lib.simopt_mv_fw_tail(sp, P(self.g), P(w_in), P(self.gamma[m:]), P(mean),
                                              self.prob.dimension, self.chunk, P(w_out),
                                              P(self.status[m:]), P(self.wmin[m:]), P(self.wsum[m:]),
                                              P(self.lin[m:]), 0 if self.prob.fused else 1))

    def _sharded_steps(self, ws, x, mean, n_k, inv):
        """Row-sharded step: exact mode gathers chunk partials (bit-identical to one
        GPU); fused mode allreduces [X_loc^T q_loc | |q_loc|^2] (d+1 doubles)."""
        lib, sp, chunk, d, sh = self.lib, _lib.stream_ptr(), self.chunk, self.prob.dimension, self.prob.shard
        P = _lib.ptr
        nl = x.shape[0]
        q = self.q[:nl]
        buf = self.red_buf
        pr = None
        if self.prob.fused and self.prob.exchange == "peer":
            from .fused import PeerReducer
            pr = PeerReducer.get(sh, d)  # collective on first use; None -> NCCL below
        for m in range(self.M):
            w_in, w_out = ws[m], ws[m + 1]
            if m == 0:
                if pr is not None:  # g summed over ranks inside the pass (peer memory)
                    fused_rows(MV, x, w_in, center=mean, col_scale=inv, col_out=self.g, peer=pr)
                elif self.prob.fused:
                    fused_rows(MV, x, w_in, center=mean, col_out=buf[:d], raw=True)
                    sh.allreduce_(buf[:d])
                    _lib.check(lib.simopt_scale_sub(sp, P(buf), inv, P(mean), d, P(self.g)))
                else:
                    if nl:
                        _lib.check(lib.simopt_matvec(sp, P(x), nl, d, None, nl, P(mean), P(w_in), chunk, P(q)))
                    sharded_matvec_t(sh, x, q, n_k, chunk, center=mean, out=self.gq)
                    _lib.check(lib.simopt_scale_sub(sp, P(self.gq), inv, P(mean), d, P(self.g)))
            _lib.check(lib.simopt_lmo_simplex_slack(sp, P(self.g), d, P(self.s), P(self.status[m:])))
            _lib.check(lib.simopt_axpy(sp, -1.0, P(w_in), P(self.s), d, P(self.dirn)))
            _lib.check(lib.simopt_axpy_ptr(sp, P(self.gamma[m:]), P(self.dirn), P(w_in), d, P(w_out)))
            _lib.check(lib.simopt_min_value(sp, P(w_out), d, P(self.wmin[m:])))
            last = m == self.M - 1
            if pr is not None:
                fused_rows(MV, x, w_out, center=mean, col_scale=inv, col_out=None if last else self.g,
                           scalar_out=self.quad[m:m + 1], accumulate=not last, peer=pr)
            elif self.prob.fused:
                fused_rows(MV, x, w_out, center=mean, col_out=None if last else buf[:d],
                           scalar_out=buf[d:], accumulate=not last, raw=True)
                if last:
                    sh.allreduce_(buf[d:])
                else:
                    sh.allreduce_(buf)
                    _lib.check(lib.simopt_scale_sub(sp, P(buf), inv, P(mean), d, P(self.g)))
                self.quad[m:m + 1].copy_(buf[d:])
            else:
                if nl:
                    _lib.check(lib.simopt_matvec(sp, P(x), nl, d, None, nl, P(mean), P(w_out), chunk, P(q)))
                sharded_dot(sh, q, q, n_k, chunk, out=self.quad[m:m + 1])
                if not last:
                    sharded_matvec_t(sh, x, q, n_k, chunk, center=mean, out=self.gq)
                    _lib.check(lib.simopt_scale_sub(sp, P(self.gq), inv, P(mean), d, P(self.g)))
            _lib.check(lib.simopt_dot(sp, P(w_out), P(mean), d, chunk, P(self.lin[m:])))
            _lib.check(lib.simopt_vec_sum(sp, P(w_out), d, chunk, P(self.wsum[m:])))
            _lib.check(lib.simopt_timestamp(sp, P(self.stamps[m:])))

    def _fused_steps(self, ws, x, mean, n_k, inv):
        lib, sp, chunk, d = self.lib, _lib.stream_ptr(), self.chunk, self.prob.dimension
        P = _lib.ptr
        for m in range(self.M):
            w_in, w_out = ws[m], ws[m + 1]
            if m == 0:  # g = (1/(N-1)) Xc^T Xc w_kM - mean
                fused_rows(MV, x, w_in, center=mean, col_scale=inv, col_out=self.g)
            self._tail(sp, m, w_in, w_out, mean)
            last = m == self.M - 1
            fused_rows(MV, x, w_out, center=mean, col_scale=inv, col_out=None if last else self.g,
                       scalar_out=self.quad[m:], accumulate=not last)
            _lib.check(lib.simopt_timestamp(sp, P(self.stamps[m:])))

    def run_epoch(self, k: int, n_k: int):
        """Enqueue epoch k's M steps on ring k % 2 (slot 0 must hold the first iterate)."""
        M = self.M
        ss = self.prob.sample_set
        x, mean = ss.samples, ss.mean
        n_rows = x.shape[0]  # this rank's rows when sharded
        if self.q is None or self.q.numel() != max(n_rows, 1):
            self.q = empty(max(n_rows, 1))
            self.graphs = {}
        ws = self.rings[k % 2]
        self.status.zero_()
        gp = self._gamma_pin[k % 2]  # its last copy (epoch k-2) ran before epoch k-1 ended
        gp.copy_(torch.tensor([fw_step_size(k, M, m) for m in range(M)], dtype=F64))
        self.gamma.copy_(gp, non_blocking=True)
        if (self.prob.fused and self.prob.shard is None and self.prob.dimension <= 2048
                and os.environ.get("SIMOPT_MV_PERSISTENT", "1") != "0"):
            # the whole epoch as one cooperative launch (simopt_mv_fw_epoch)
            P = _lib.ptr
            _lib.check(self.lib.simopt_mv_fw_epoch(
                _lib.stream_ptr(), P(x), n_k, self.prob.dimension, P(mean), 1.0 / (n_k - 1), P(ws), M,
                P(self.gamma), P(self.status), P(self.wmin), P(self.wsum), P(self.lin), P(self.quad),
                P(self.stamps)))
            return
        key = (k % 2, x.data_ptr(), mean.data_ptr(), n_k, self.prob.fused)
        g = self.graphs.get(key)
        if not self.use_graph or self.prob.shard is not None:  # collectives: eager
            self._steps(ws, x, mean, n_k)
            return
        if g is None and not self.warm:
            # first epoch eager on the capture stream: lazy library setup and the
            # stream's scratch happen outside any capture
            self.cstream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.cstream):
                self._steps(ws, x, mean, n_k)
            torch.cuda.current_stream().wait_stream(self.cstream)
            self.warm = True
            return
        if g is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.cstream):
                self._steps(ws, x, mean, n_k)
            self.graphs[key] = g
        g.replay()


def _mv_fw_run_device(prob: MeanVarProblem, config, backend, label, size, rep):
    M, K = config.inner_iters, config.epochs
    T = K * M
    eng = prob._engines.get((M, backend.chunk_size, prob.fused))
    if eng is None:  # kept on the problem: its captured epoch graphs are reused by later runs
        eng = prob._engines[(M, backend.chunk_size, prob.fused)] = MvFwEngine(prob, M, backend.chunk_size)
    eng.rings[0][0].zero_()
    status = torch.zeros(T, dtype=torch.int32, device="cuda")
    wmin, wsum, quad, lin = empty(T), empty(T), empty(T), empty(T)
    stamps = torch.zeros(T + 1, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    _lib.check(lib.simopt_timestamp(_lib.stream_ptr(), _lib.ptr(stamps[T:])))
    trace = TraceBuilder()
    n_of, events, host = [], [], {}
    # epoch records are read back on a side stream into pinned buffers, ordered after their
    # epoch only: a plain device-to-host copy on the main stream would also wait for the
    # epoch enqueued after it and leave the GPU idle while the host enqueues the next one
    rd_stream = torch.cuda.Stream()
    pins = [torch.empty(M, dtype=a.dtype, pin_memory=True) for a in (status, wmin, wsum, quad, lin, stamps)]
    t0_pin = torch.empty(1, dtype=torch.int64, pin_memory=True)

    def check_epoch(k):
        """Host validation of epoch k (its ring is intact until epoch k+2 is enqueued)."""
        sl = slice(k * M, (k + 1) * M)
        with torch.cuda.stream(rd_stream):
            rd_stream.wait_event(events[k])
            for pin, a in zip(pins, (status, wmin, wsum, quad, lin, stamps)):
                pin.copy_(a[sl], non_blocking=True)
            if k == 0:
                t0_pin.copy_(stamps[T:], non_blocking=True)
            got = torch.cuda.Event()
            got.record(rd_stream)
        got.synchronize()
        if prob.shard is not None and prob.fused and prob.exchange == "peer":
            from .fused import PeerReducer
            pr = PeerReducer.get(prob.shard, prob.dimension)
            if pr is not None:
                pr.check()
        st, mn, sm, qd, ln, ts = (pin.numpy() for pin in pins)
        t0 = host.setdefault("t0", int(t0_pin[0]))
        ws = eng.rings[k % 2]
        for m in range(M):
            t = k * M + m
            if st[m] != 0:
                return InvalidGradient("gradient contains NaN"), ws[m]
            if not (mn[m] >= -FEAS_TOL and sm[m] <= 1.0 + FEAS_TOL):
                return InvalidConstraint(f"iterate infeasible at step {t + 1}"), ws[m + 1]
            f = 0.5 * float(qd[m]) / (n_of[k] - 1) - float(ln[m])  # tasks.py:75
            trace.append(t + 1, f, int(ts[m]) - t0)
        return None

    def abort(exc, it):
        partial = trace.build(label, size, backend.kind, rep, config.stream.seed, to_host(it))
        raise RunAborted(f"frank-wolfe run failed at step {len(trace) + 1}: {exc}", partial) from exc

    # Double-buffered epochs (unsharded diagonal model, when two copies of X fit): epoch
    # k+1's draw runs on a low-priority stream into the other buffer while epoch k's
    # HBM-bound steps run -- the exact glibc normals are FP64/INT-issue-bound, so the two
    # overlap instead of adding up.  The draws keep the sequential stream order.
    sizes = [config.epoch_sample_size(k) for k in range(K)]
    nbytes = 8 * max(sizes) * prob.dimension
    pipelined = (prob.shard is None and prob.task.spec.diag_std is not None and K > 1
                 and 2 * nbytes < 0.4 * torch.cuda.get_device_properties(0).total_memory)
    main = torch.cuda.current_stream()
    if pipelined:
        lo_pri = torch.cuda.Stream.priority_range()[0] if hasattr(torch.cuda.Stream, "priority_range") else 0
        gen = eng.gen_stream = getattr(eng, "gen_stream", None) or torch.cuda.Stream(priority=lo_pri)
        sets, ready, steps_done = {}, {}, {}
        start = torch.cuda.Event()
        start.record(main)  # the run's setup; slot 1 is free before epoch 0's steps end

        def draw(k):
            slot = k % 2
            gen.wait_event(start if k < 2 else steps_done[k - 2])  # last reader of the slot
            with torch.cuda.stream(gen):
                sets[k] = prob.resample_slot(config.stream, sizes[k], slot)
                ev = torch.cuda.Event()
                ev.record()
            ready[k] = ev
        draw(0)
    for k in range(K):
        n_k = sizes[k]
        n_of.append(n_k)
        if k >= 1:
            eng.rings[k % 2][0].copy_(eng.rings[(k - 1) % 2][M])  # roll the iterate
        if pipelined:
            main.wait_event(ready.pop(k))
            prob.sample_set = sets.pop(k)
            eng.run_epoch(k, n_k)
            done = torch.cuda.Event()
            done.record(main)
            steps_done[k] = done
            if k + 1 < K:
                draw(k + 1)
        else:
            prob.resample(config.stream, n_k)
            eng.run_epoch(k, n_k)
        sl = slice(k * M, (k + 1) * M)
        for dst, src in ((status, eng.status), (wmin, eng.wmin), (wsum, eng.wsum),
                         (quad, eng.quad), (lin, eng.lin), (stamps, eng.stamps)):
            dst[sl].copy_(src)
        ev = torch.cuda.Event()
        ev.record()
        events.append(ev)
        if k >= 1:  # validate the previous epoch while this one runs
            bad = check_epoch(k - 1)
            if bad:
                abort(*bad)
    bad = check_epoch(K - 1)
    if bad:
        abort(*bad)
    return trace.build(label, size, backend.kind, rep, config.stream.seed,
                       to_host(eng.rings[(K - 1) % 2][M]))


# ---------------------------------------------------------------------------
# Task 3: binary classification (logistic loss), tasks.py:196-253
@dataclass
class LogisticTask:
    data: "ClassificationData"

    @property
    def dimension(self) -> int:
        return self.data.n_features


def _batch_rows(data, indices):
    """tasks.py:205-213 without the row copy: a device index vector for the gather."""
    if indices is None:
        return None, data.n_samples
    idx = indices if is_tensor(indices) else torch.as_tensor(np.asarray(indices), dtype=torch.int64)
    idx = idx.to(device="cuda", dtype=torch.int64).contiguous()
    if idx.numel() == 0:
        raise ConfigurationError("empty index set")
    if int(idx.min().item()) < 0 or int(idx.max().item()) >= data.n_samples:
        raise ConfigurationError("batch index out of range")
    return idx, idx.numel()


def x_matvec(data, backend, v, idx=None, out=None) -> torch.Tensor:
    """Fixed-tree X_b v over this rank's rows (gathered through idx); bit-packed features
    are read as bits (simopt_matvec_bits_idx, bit-identical to the 0/1 fp64 matrix)."""
    if not data.packed:
        return backend.matvec_device(data.features, v, out=out, rows_idx=idx)
    if v.numel() != data.n_features:
        raise DimensionMismatch(f"matvec: ({data.local_rows}, {data.n_features}) @ ({v.numel()},)")
    rows = data.local_rows if idx is None else idx.numel()
    out = empty(rows) if out is None else out
    _lib.call("simopt_matvec_bits_idx", _lib.stream_ptr(), _lib.ptr(data.bits), data.local_rows,
              data.n_features, _lib.ptr(idx), rows, _lib.ptr(v), backend.chunk_size, _lib.ptr(out))
    return out


def x_matvec_t(data, backend, x, idx=None, out=None) -> torch.Tensor:
    """Fixed-tree X_b^T x (column sums over the gathered rows); bits when packed."""
    if not data.packed:
        return backend.matvec_t_device(data.features, x, out=out, rows_idx=idx)
    rows = data.local_rows if idx is None else idx.numel()
    if x.numel() != rows:
        raise DimensionMismatch(f"matvec_t: ({rows}, {data.n_features})^T @ ({x.numel()},)")
    out = empty(data.n_features) if out is None else out
    _lib.call("simopt_matvec_t_bits", _lib.stream_ptr(), _lib.ptr(data.bits), data.local_rows,
              data.n_features, _lib.ptr(idx), rows, _lib.ptr(x), backend.chunk_size, _lib.ptr(out))
    return out


def logistic_loss_device(w, data, indices, backend, idx=None, out=None) -> torch.Tensor:
    """Device scalar sum of logistic_loss_block terms (divide by the batch size on read)."""
    wd = vec_dev(w)
    if wd.numel() != data.n_features:
        raise DimensionMismatch("weight length != feature count")
    if idx is None:
        idx, b = _batch_rows(data, indices)
    else:
        b = idx.numel()
    t = x_matvec(data, backend, wd, idx)
    terms = empty(b)
    _lib.call("simopt_logistic_loss_terms", _lib.stream_ptr(), _lib.ptr(t), _lib.ptr(data.labels),
              _lib.ptr(idx), b, _lib.ptr(terms))
    return backend.vec_sum_device(terms, out=out)


def logistic_loss(w, data, indices, backend) -> float:
    """Mean negative log-likelihood over the given rows (tasks.py:216-225)."""
    idx, b = _batch_rows(data, indices)
    s = logistic_loss_device(w, data, indices, backend, idx=idx)
    return float(s.item()) / b


def logistic_gradient_device(w, data, indices, backend, idx=None, out=None) -> torch.Tensor:
    """(1/b) X_b^T (c - z_b) with exact trees (tasks.py:228-236)."""
    wd = vec_dev(w)
    if wd.numel() != data.n_features:
        raise DimensionMismatch("weight length != feature count")
    if idx is None:
        idx, b = _batch_rows(data, indices)
    else:
        b = idx.numel()
    t = x_matvec(data, backend, wd, idx)
    r = empty(b)
    _lib.call("simopt_logistic_resid", _lib.stream_ptr(), _lib.ptr(t), _lib.ptr(data.labels),
              _lib.ptr(idx), b, _lib.ptr(r))
    gt = x_matvec_t(data, backend, r, idx)
    out = empty(gt.numel()) if out is None else out
    _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(gt), 1.0 / b, None, gt.numel(),
              _lib.ptr(out))
    return out


def logistic_gradient(w, data, indices, backend):
    return like_input(w, logistic_gradient_device(w, data, indices, backend))


def logistic_hvp_device(w, v, data, indices, backend, idx=None, out=None) -> torch.Tensor:
    """Sub-sampled Hessian-vector product (1/b) X_b^T diag(c(1-c)) X_b v (tasks.py:239-253)."""
    wd, vd = vec_dev(w), vec_dev(v)
    if wd.numel() != data.n_features or vd.numel() != data.n_features:
        raise DimensionMismatch("vector length != feature count")
    if idx is None:
        idx, b = _batch_rows(data, indices)
    else:
        b = idx.numel()
    t = x_matvec(data, backend, wd, idx)
    tv = x_matvec(data, backend, vd, idx)
    wt = empty(b)
    _lib.call("simopt_logistic_hvp_weights", _lib.stream_ptr(), _lib.ptr(t), _lib.ptr(tv), b,
              _lib.ptr(wt))
    ht = x_matvec_t(data, backend, wt, idx)
    out = empty(ht.numel()) if out is None else out
    _lib.call("simopt_scale_sub", _lib.stream_ptr(), _lib.ptr(ht), 1.0 / b, None, ht.numel(),
              _lib.ptr(out))
    return out


def logistic_hvp(w, v, data, indices, backend):
    return like_input(w, logistic_hvp_device(w, v, data, indices, backend))
