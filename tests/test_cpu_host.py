"""CPU-only checks: ABI exports, host-side logic, error mapping, sharding (gloo, world_size 2)."""
import ctypes
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_abi_exports_every_declared_symbol():
    from paper_2404_11631_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2404_11631_b200 import build
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    header = open(os.path.join(ROOT, "include", "simopt_b200.h")).read()
    declared = set(re.findall(r"\b(simopt_\w+)\s*\(", header))
    assert declared, "no declarations parsed"
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.exported_symbols()) <= declared
    lib.simopt_abi_version.restype = ctypes.c_int
    assert lib.simopt_abi_version() == _lib.ABI_VERSION


def test_no_device_means_loud_failure(monkeypatch):
    import paper_2404_11631_b200 as pkg
    from paper_2404_11631_b200 import _lib
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(pkg.DeviceError):
        _lib.load()


def test_status_codes_map_to_reference_errors():
    from paper_2404_11631_b200 import errors as e
    assert e.STATUS_TO_ERROR[1] is e.DimensionMismatch and issubclass(e.DimensionMismatch, ValueError)
    assert e.STATUS_TO_ERROR[2] is e.ConfigurationError
    assert e.STATUS_TO_ERROR[5] is e.InvalidGradient
    assert e.STATUS_TO_ERROR[8] is e.DegeneratePair
    assert issubclass(e.RunAborted, RuntimeError)


def test_rng_stream_semantics():
    from paper_2404_11631_b200 import ConfigurationError, RngStream
    s = RngStream(42, 7, (1 << 64) + 5)
    assert s.words() == (42, 7, 5, 1)
    s.advance(9)
    assert s.counter == (1 << 64) + 5 + 3
    assert s.clone() == s and s.clone() is not s
    with pytest.raises(ConfigurationError):
        RngStream(-1, 0)
    with pytest.raises(ConfigurationError):
        RngStream(0, 1 << 64)


def test_fw_config_and_step_size():
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_step_size
    from paper_2404_11631_b200 import ConfigurationError, RngStream
    assert fw_step_size(0, 25, 0) == 1.0
    assert fw_step_size(3, 25, 4) == 2.0 / (3 * 25 + 4 + 2)
    with pytest.raises(ConfigurationError):
        fw_step_size(0, 5, 5)
    with pytest.raises(ConfigurationError):
        FwConfig(0, 1, 1, RngStream(1, 1))
    assert FwConfig(2, 3, 10, RngStream(1, 1), "linear").epoch_sample_size(2) == 30


def test_task_validation():
    from paper_2404_11631_b200.tasks import NewsvendorTask
    from paper_2404_11631_b200 import InvalidConstraint, ConfigurationError, DimensionMismatch
    ok = dict(unit_cost=[1.0, 1.5], holding_cost=[0.5, 0.6], selling_value=[3.0, 4.0],
              demand_mean=[20.0, 30.0], demand_std=[10.0, 11.0], budget_costs=[1.0, 1.0], budget=25.0)
    NewsvendorTask(**ok)
    with pytest.raises(InvalidConstraint):
        NewsvendorTask(**{**ok, "unit_cost": [5.0, 1.0]})
    with pytest.raises(DimensionMismatch):
        NewsvendorTask(**{**ok, "demand_std": [1.0]})
    with pytest.raises(ConfigurationError):
        NewsvendorTask(**{**ok, "budget": None})


def test_make_backend_rejects_gpu_kind():
    from paper_2404_11631_b200 import ConfigurationError, make_backend
    with pytest.raises(ConfigurationError):
        make_backend("gpu")
    with pytest.raises(ConfigurationError):
        make_backend("cuda", chunk_size=0)


def test_shard_range_and_blocks():
    from paper_2404_11631_b200.sharding import first_block, shard_range
    d = 10_000
    spans = [shard_range(d, 3, r) for r in range(3)]
    assert spans[0][0] == 0 and spans[-1][1] == d
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert all(lo % 4096 == 0 for lo, _ in spans)
    assert first_block(3, 100_000) == (75_000, 0)
    assert first_block(1, 7) == (1, 3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, x, y, want, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_11631_b200.sharding import allgather_fold, allreduce_argmin, shard_range
    lo, hi = shard_range(x.size, world, rank)
    partials = [orc.dot(x[c:min(c + 4096, hi)], y[c:min(c + 4096, hi)]) for c in range(lo, hi, 4096)]
    root = allgather_fold(torch.tensor(partials, dtype=torch.float64))
    g = x * y
    j = lo + int(np.argmin(g[lo:hi]))
    best = allreduce_argmin(float(g[j]), j)
    q.put((rank, root, best))
    dist.destroy_process_group()


def test_gloo_sharded_exact_tree_and_argmin():
    """World-size-2 sharded reduction folds to the single-process tree bitwise."""
    rng = np.random.default_rng(3)
    n = 3 * 4096 + 777
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    want = orc.dot(x, y)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, y, want, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    g = x * y
    for _, root, best in res:
        assert root == want
        assert best == (float(g[int(np.argmin(g))]), int(np.argmin(g)))


def _group_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_11631_b200.sharding import ShardGroup
    sh = ShardGroup()
    t = torch.full((3,), float(rank + 1), dtype=torch.float64)
    sh.allreduce_(t)
    g = sh.allgather(torch.tensor([rank, 10 * rank], dtype=torch.float64))
    lo, hi = sh.range(10, 4)
    rows = torch.arange(lo, hi, dtype=torch.float64).view(-1, 1)
    cat = sh.allgather_rows(rows, [b - a for a, b in sh.ranges(10, 4)])
    q.put((rank, t.tolist(), g.tolist(), cat.view(-1).tolist(), (lo, hi)))
    dist.destroy_process_group()


def test_gloo_shard_group_collectives():
    """ShardGroup (the sharded solvers' only communication layer) over gloo, world 2."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_group_worker, args=(r, 2, port, q)) for r in range(3 - 1)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, t, g, cat, rng in res:
        assert t == [3.0, 3.0, 3.0]
        assert g == [[0.0, 0.0], [1.0, 10.0]]
        assert cat == [float(i) for i in range(10)]      # uneven shards [0,8) and [8,10)
    assert res[0][4] == (0, 8) and res[1][4] == (8, 10)


def test_shifted_counter_matches_block_offset():
    """A product shard's draw = the full draw with the counter moved by whole blocks."""
    from paper_2404_11631_b200.sharding import shifted_counter
    S, j0 = 5000, 504
    full = orc.standard_normal(orc.Stream(42, 2), 1003 * S)
    st = orc.Stream(42, 2)
    st.counter = shifted_counter(0, j0 * S // 4)
    part = orc.standard_normal(st, 8 * S)
    assert np.array_equal(part, full[j0 * S:(j0 + 8) * S])
    assert shifted_counter((1 << 128) - 1, 2) == 1


def test_product_sharding_rejects_empty_ranks():
    """Every rank must own products (each step's LMO exchange waits for all ranks): a
    product count that leaves a rank empty is rejected up front, not a 10 s exchange timeout."""
    import numpy as np
    import paper_2404_11631_b200 as p
    from paper_2404_11631_b200.sharding import shard_range
    from paper_2404_11631_b200.tasks import NewsvendorProblem, NewsvendorTask

    class Shard:  # the ShardGroup interface NewsvendorProblem uses before touching the GPU
        world, rank = 8, 0

        def range(self, n, align=1):
            return shard_range(n, self.world, self.rank, align)

        def ranges(self, n, align=1):
            return [shard_range(n, self.world, r, align) for r in range(self.world)]

    task = NewsvendorTask(unit_cost=np.full(10, 1.5), holding_cost=np.full(10, 0.7),
                          selling_value=np.full(10, 4.0), demand_mean=np.full(10, 30.0),
                          demand_std=np.full(10, 15.0), budget_costs=np.ones(10), budget=150.0)
    with pytest.raises(p.ConfigurationError):
        NewsvendorProblem(task, None, shard=Shard())
