"""Sharded solver runs vs the one-process oracle, world size 2 on one GPU.

Two ranks share cuda:0 over gloo, which exercises every sharded code path
(row-shard RNG addressing, chunk-partial gathers, fused allreduces, the product
-sharded LMO exchange) except NCCL itself.  Exact-tree modes must be bit-identical
to the single-process oracle; fused modes within the north-star 1e-8.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def ranks(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("sharded"))
    port = _port()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_sharded_worker.py"), str(r), "2",
                               str(port), out]) for r in range(2)]
    for pr in procs:
        assert pr.wait(timeout=600) == 0
    return [dict(np.load(os.path.join(out, f"rank{r}.npz"))) for r in range(2)]


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_ranks_agree(ranks):
    a, b = ranks
    for k in a:
        if k != "lr_rows":
            assert np.array_equal(a[k], b[k]), k
    assert a["lr_rows"][0] + b["lr_rows"][0] == 9000 and b["lr_rows"][1] == a["lr_rows"][0]


@pytest.mark.parametrize("chunk", [4096, 1000])
def test_meanvar_sharded(ranks, chunk):
    mu, sigma = orc.gen_meanvar_instance(300, orc.Stream(42, 0))
    objs, w = orc.fw_run_meanvar(mu, sigma, 2, 10, 10_000, orc.Stream(42, 2), chunk)
    r = ranks[0]
    assert np.array_equal(r[f"mv_{chunk}_0_obj"], objs)      # exact tree: bitwise
    assert np.array_equal(r[f"mv_{chunk}_0_w"], w)
    for mode in (1, 2):                                       # fused: peer-memory / NCCL sums
        np.testing.assert_allclose(r[f"mv_{chunk}_{mode}_obj"], objs, rtol=1e-8)
        assert _rel(r[f"mv_{chunk}_{mode}_w"], w) < 1e-8


def test_logistic_sharded(ranks):
    x, z, _ = orc.synth_classification(40, orc.Stream(42, 0), n_rows=9000)
    objs, w = orc.newton_cg(x, z, iterations=3, cg_iters=8)
    r = ranks[0]
    assert np.array_equal(r["ncg_0_obj"], objs)
    assert np.array_equal(r["ncg_0_w"], w)
    assert bool(r["peer_reduce_used"][0])                    # the in-kernel peer allreduce ran
    for mode in (1, 2):
        np.testing.assert_allclose(r[f"ncg_{mode}_obj"], objs, rtol=1e-8)
        assert _rel(r[f"ncg_{mode}_w"], w) < 1e-8
    np.testing.assert_allclose(r["ncgp_obj"], objs, rtol=1e-8)      # bit-packed shards
    assert _rel(r["ncgp_w"], w) < 1e-8
    objs, w = orc.newton_explicit(x, z, iterations=3, cg_iters=20)
    np.testing.assert_allclose(r["nex_obj"], objs, rtol=1e-8)
    assert _rel(r["nex_w"], w) < 1e-8
    np.testing.assert_allclose(r["nexp_obj"], objs, rtol=1e-8)
    assert _rel(r["nexp_w"], w) < 1e-8
    # d = 1100 > 1024: the banded two-sweep bit-packed passes, cross-rank sums in peer memory
    x, z, _ = orc.synth_classification(1100, orc.Stream(42, 0), n_rows=3000)
    objs, w = orc.newton_cg(x, z, iterations=2, cg_iters=4)
    np.testing.assert_allclose(r["ncgw_obj"], objs, rtol=1e-8)
    assert _rel(r["ncgw_w"], w) < 1e-8


def test_newsvendor_sharded(ranks):
    task = orc.gen_newsvendor_instance(1003, orc.Stream(42, 0))
    objs, x = orc.fw_run_newsvendor(task, 5, 6, 5000, orc.Stream(42, 2))  # epochs 2+ replay graphs
    r = ranks[0]
    assert bool(r["nv_peer_used"][0])                      # the in-kernel NVLink/IPC exchange ran
    for ex in ("nccl", "peer"):
        assert np.array_equal(r[f"nv_{ex}_w"], x)          # counts are exact integers
        np.testing.assert_allclose(r[f"nv_{ex}_obj"], objs, rtol=1e-13)
    objs, x = orc.fw_run_newsvendor(task, 5, 4, 2000, orc.Stream(42, 2), schedule="linear")
    assert np.array_equal(r["nv_lin_w"], x)
    np.testing.assert_allclose(r["nv_lin_obj"], objs, rtol=1e-13)


def test_full_size_sharded(ranks, golden):
    """BASELINE sizes with two ranks: C2 (products, peer-memory LMO, graph epochs) and the
    exact C3/C4 modes bit for bit vs the reference's trajectories; fused within 1e-8."""
    r = ranks[0]
    g = golden("full_c2")
    assert np.array_equal(r["full_c2_w"], g["final_iterate"])
    # the recorded objective sums the two shards' exact-tree sums (not the reference's
    # one 4096-chunk tree over all d products): last-bit differences only
    np.testing.assert_allclose(r["full_c2_obj"], g["objectives"], rtol=1e-13)
    g = golden("full_c4")
    assert np.array_equal(r["full_c4_0_obj"], g["objectives"])
    assert np.array_equal(r["full_c4_0_w"], g["final_iterate"])
    np.testing.assert_allclose(r["full_c4_1_obj"], g["objectives"], rtol=1e-8)
    assert _rel(r["full_c4_1_w"], g["final_iterate"]) < 1e-8
    g = golden("full_c3")
    assert np.array_equal(r["full_c3_0_obj"], g["objectives"])
    assert np.array_equal(r["full_c3_0_w"], g["final_iterate"])
    np.testing.assert_allclose(r["full_c3_1_obj"], g["objectives"], rtol=1e-8)
    assert _rel(r["full_c3_1_w"], g["final_iterate"]) < 1e-8


def test_simopt_comm_world1():
    """The C-ABI NCCL communicator (simopt_comm_*): a one-rank communicator's all-reduce and
    all-gather are the identity (a multi-rank NCCL group needs one GPU per rank)."""
    import torch
    from paper_2404_11631_b200.sharding import SimoptComm
    c = SimoptComm(0, 1)
    x = torch.arange(10, dtype=torch.float64, device="cuda")
    assert torch.equal(c.allreduce_(x.clone()), x)
    assert torch.equal(c.allgather(x)[0], x)
    c.close()
