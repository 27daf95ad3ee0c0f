"""Small instances of the kernels with hand-rolled synchronisation, for compute-sanitizer.

  compute-sanitizer --tool {memcheck|racecheck|synccheck} python tools/sanitize_paths.py PATH
  PATH: nv         newsvendor resample (warp-specialised, named barriers) + fused FW steps
                   (last-block reduction, dynamic product counter) + recording sums
        fused      mean-variance / logistic fused row passes, every cluster width (st.async
                   DSMEM exchange on mbarriers), dense and bit-packed X; the persistent
                   mean-variance epoch (cooperative grid barriers)
        hessian    limb Hessians: tcgen05 cp.async (tc), TMA + mbarrier ring (tma), CTA pair
        peer RANK WORLD PORT  one rank of a product-sharded newsvendor run and a sharded fused
                   mean-variance run whose sums cross ranks over CUDA-IPC peer mailboxes
                   (release/acquire flags); start one process per rank
Every path checks its results against a reference computed another way, so a run that
"passes" the sanitizer also produced the right numbers under it.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_11631_b200 as p  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def nv():
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    b = p.make_backend("cuda")
    # d = 37 products; S = 9001: three 4096-segments, the last ragged, rows not 4-aligned
    # (scalar key loads); S = 8192: aligned rows (16-byte key loads)
    for d, S, K, M in ((37, 9001, 2, 3), (37, 8192, 2, 3)):
        rec = fw_run(NewsvendorProblem(gen_newsvendor_instance(d, p.RngStream(42, 0)), b),
                     FwConfig(K, M, S, p.RngStream(42, 2)), b)
        task = orc.gen_newsvendor_instance(d, orc.Stream(42, 0))
        objs, x = orc.fw_run_newsvendor(task, K, M, S, orc.Stream(42, 2))
        assert np.array_equal(rec.final_iterate, x), f"iterate differs from the oracle (S={S})"
        assert np.allclose(rec.objectives, objs, rtol=1e-13, atol=0)
    print("nv ok")


def fused():
    from paper_2404_11631_b200.fused import LR_GRAD, MV, fused_rows
    rng = np.random.default_rng(0)
    for n, d in [(97, 20000), (300, 8192), (200, 2500), (777, 7)]:  # cluster widths 8, 4, 2, 1
        x = rng.standard_normal((n, d))
        v = rng.standard_normal(d) * 0.1
        mean = rng.standard_normal(d) * 0.01
        X, V, Mn = (torch.from_numpy(a).cuda() for a in (x, v, mean))
        g = torch.empty(d, dtype=torch.float64, device="cuda")
        sc = torch.empty(1, dtype=torch.float64, device="cuda")
        fused_rows(MV, X, V, center=Mn, col_scale=1.0, col_out=g, scalar_out=sc)
        q = (x - mean) @ v
        want = (x - mean).T @ q - mean
        assert np.linalg.norm(g.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want), (n, d)
        z = torch.from_numpy((rng.random(n) < 0.5).astype(float)).cuda()
        fused_rows(LR_GRAD, X, V, rowaux=z, col_scale=1.0 / n, col_out=g, scalar_out=sc)
        c = orc.sigmoid(x @ v)
        want = x.T @ (c - z.cpu().numpy()) / n
        assert np.linalg.norm(g.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want), (n, d)
    from paper_2404_11631_b200.newton import newton_cg
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.tasks import LogisticTask
    b = p.make_backend("cuda")
    for d, n in [(1000, 3000), (2000, 1500)]:  # nibble-table passes, banded for d > 1024
        dense = synth_classification(d, p.RngStream(5, 0), n_rows=n)
        packed = synth_classification(d, p.RngStream(5, 0), n_rows=n, packed=True)
        r0 = newton_cg(LogisticTask(dense), 2, 4, b, fused=True)
        r1 = newton_cg(LogisticTask(packed), 2, 4, b, fused=True)
        np.testing.assert_allclose(r1.objectives, r0.objectives, rtol=1e-8)  # fused: north-star 1e-8
    # the persistent mean-variance epoch (cooperative launch, grid barriers, redundant tails):
    # warp-per-row (d = 300) and CTA-per-row (d = 1500) passes against the launch sequence
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    for d, n in [(300, 2000), (1500, 1200)]:
        task = gen_meanvar_instance(d, p.RngStream(42, 0))
        recs = []
        for flag in ("1", "0"):
            os.environ["SIMOPT_MV_PERSISTENT"] = flag
            recs.append(fw_run(MeanVarProblem(task, b, fused=True), FwConfig(2, 5, n, p.RngStream(42, 2)), b))
        os.environ.pop("SIMOPT_MV_PERSISTENT")
        np.testing.assert_allclose(recs[0].objectives, recs[1].objectives, rtol=1e-10)
    print("fused ok")


def hessian():
    from paper_2404_11631_b200.newton import logistic_hessian_device
    from paper_2404_11631_b200.sampling import synth_classification
    for d, n in [(256, 5000), (130, 64), (200, 3001)]:
        data = synth_classification(d, p.RngStream(8, 0), n_rows=n, packed=True)
        dw = torch.rand(n, dtype=torch.float64, device="cuda") * 0.25
        ref = logistic_hessian_device(data, dw, method="dmma")
        for m in ("tc", "tma", "pair"):
            got = logistic_hessian_device(data, dw, method=m)
            err = ((got - ref).abs().max() / ref.abs().max()).item()
            assert err < 1e-10, (m, d, n, err)
    print("hessian ok")


def peer(rank, world, port):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), LOCAL_RANK="0")
    import torch.distributed as dist
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.sharding import ShardGroup
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    shard = ShardGroup()
    b = p.make_backend("cuda")
    d, S, K, M = 64, 5000, 2, 3
    prob = NewsvendorProblem(gen_newsvendor_instance(d, p.RngStream(42, 0)), b, shard=shard)
    rec = fw_run(prob, FwConfig(K, M, S, p.RngStream(42, 2)), b)
    task = orc.gen_newsvendor_instance(d, orc.Stream(42, 0))
    objs, x = orc.fw_run_newsvendor(task, K, M, S, orc.Stream(42, 2))
    assert np.array_equal(rec.final_iterate, x), "sharded iterate differs from the oracle"
    assert np.allclose(rec.objectives, objs, rtol=1e-13, atol=0)
    from paper_2404_11631_b200.tasks import MeanVarProblem
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    mv = gen_meanvar_instance(300, p.RngStream(42, 0))
    prob = MeanVarProblem(mv, b, fused=True, shard=shard)
    rec = fw_run(prob, FwConfig(2, 5, 4000, p.RngStream(42, 2)), b)
    mu, sigma = orc.gen_meanvar_instance(300, orc.Stream(42, 0))
    objs, w = orc.fw_run_meanvar(mu, sigma, 2, 5, 4000, orc.Stream(42, 2), 4096)
    np.testing.assert_allclose(rec.objectives, objs, rtol=1e-8)
    dist.barrier()
    dist.destroy_process_group()
    print(f"peer rank {rank} ok")


if __name__ == "__main__":
    what = sys.argv[1]
    if os.environ.get("SANITIZE_PREINIT"):
        torch.zeros(1, device="cuda")  # the runtime's context is current before the library's first launch
    if what == "peer":
        peer(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
    else:
        {"nv": nv, "fused": fused, "hessian": hessian}[what]()
    torch.cuda.synchronize()
