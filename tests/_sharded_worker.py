"""Child process of tests/test_gpu_sharded.py: one rank of a sharded solver run.

Ranks share cuda:0 and talk over gloo (the one-GPU box); on a multi-GPU box the
same code runs one rank per GPU over NCCL.  Each rank writes its RunRecords to
<out>/rank<r>.npz for the parent to compare against the oracle.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(rank, world, port, out):
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2404_11631_b200 as p
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_meanvar_instance, gen_newsvendor_instance
    from paper_2404_11631_b200.newton import newton_cg, newton_explicit
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.sharding import ShardGroup
    from paper_2404_11631_b200.tasks import LogisticTask, MeanVarProblem, NewsvendorProblem
    sh = ShardGroup()
    res = {}
    for chunk in (4096, 1000):
        b = p.make_backend("cuda", chunk_size=chunk)
        for fused in (False, True):
            task = gen_meanvar_instance(300, p.RngStream(42, 0))
            rec = fw_run(MeanVarProblem(task, b, fused=fused, shard=sh),
                         FwConfig(2, 10, 10_000, p.RngStream(42, 2)), b)
            res[f"mv_{chunk}_{int(fused)}_obj"] = rec.objectives
            res[f"mv_{chunk}_{int(fused)}_w"] = rec.final_iterate
        task = gen_meanvar_instance(300, p.RngStream(42, 0))  # fused, NCCL/gloo allreduce path
        rec = fw_run(MeanVarProblem(task, b, fused=True, shard=sh, exchange="nccl"),
                     FwConfig(2, 10, 10_000, p.RngStream(42, 2)), b)
        res[f"mv_{chunk}_2_obj"], res[f"mv_{chunk}_2_w"] = rec.objectives, rec.final_iterate
    b = p.make_backend("cuda")
    data = synth_classification(40, p.RngStream(42, 0), n_rows=9000, shard=sh)
    res["lr_rows"] = np.array([data.local_rows, data.row_offset])
    for fused in (False, True):
        rec = newton_cg(LogisticTask(data), 3, 8, b, fused=fused)
        res[f"ncg_{int(fused)}_obj"] = rec.objectives
        res[f"ncg_{int(fused)}_w"] = rec.final_iterate
    rec = newton_cg(LogisticTask(data), 3, 8, b, exchange="nccl")
    res["ncg_2_obj"], res["ncg_2_w"] = rec.objectives, rec.final_iterate
    from paper_2404_11631_b200.fused import PeerReducer
    res["peer_reduce_used"] = np.array([PeerReducer.get(sh, 40) is not None])
    rec = newton_explicit(LogisticTask(data), 3, 20, b)
    res["nex_obj"], res["nex_w"] = rec.objectives, rec.final_iterate
    packed = synth_classification(40, p.RngStream(42, 0), n_rows=9000, shard=sh, packed=True)
    rec = newton_cg(LogisticTask(packed), 3, 8, b)
    res["ncgp_obj"], res["ncgp_w"] = rec.objectives, rec.final_iterate
    rec = newton_explicit(LogisticTask(packed), 3, 20, b)
    res["nexp_obj"], res["nexp_w"] = rec.objectives, rec.final_iterate
    wide = synth_classification(1100, p.RngStream(42, 0), n_rows=3000, shard=sh, packed=True)
    rec = newton_cg(LogisticTask(wide), 2, 4, b)   # banded nibble passes (d > 1024), peer sums
    res["ncgw_obj"], res["ncgw_w"] = rec.objectives, rec.final_iterate
    nv = gen_newsvendor_instance(1003, p.RngStream(42, 0))
    for ex in ("nccl", "peer"):
        rec = fw_run(NewsvendorProblem(nv, b, shard=sh, exchange=ex),
                     FwConfig(5, 6, 5000, p.RngStream(42, 2)), b)
        res[f"nv_{ex}_obj"], res[f"nv_{ex}_w"] = rec.objectives, rec.final_iterate
    # a linear sample schedule: S (and the layout slots) change every epoch, so the
    # graph engine must re-capture per layout (stale captured S/keys)
    rec = fw_run(NewsvendorProblem(nv, b, shard=sh, exchange="peer"),
                 FwConfig(5, 4, 2000, p.RngStream(42, 2), "linear"), b)
    res["nv_lin_obj"], res["nv_lin_w"] = rec.objectives, rec.final_iterate
    # BASELINE sizes (tests/golden/full_*.npz): C2 products sharded, graph engine + peer LMO
    nvf = gen_newsvendor_instance(10_000, p.RngStream(42, 0))
    rec = fw_run(NewsvendorProblem(nvf, b, shard=sh), FwConfig(3, 25, 100_000, p.RngStream(42, 2)), b)
    res["full_c2_obj"], res["full_c2_w"] = rec.objectives, rec.final_iterate
    del nvf
    for fused in (False, True):  # C4's d at N = 2*10^4, rows sharded
        mvf = gen_meanvar_instance(20_000, p.RngStream(42, 0))
        rec = fw_run(MeanVarProblem(mvf, b, fused=fused, shard=sh),
                     FwConfig(1, 25, 20_000, p.RngStream(42, 2)), b)
        res[f"full_c4_{int(fused)}_obj"], res[f"full_c4_{int(fused)}_w"] = rec.objectives, rec.final_iterate
    big = synth_classification(1_000, p.RngStream(42, 0), n_rows=1_000_000, shard=sh, packed=True)
    for fused in (False, True):  # C3 rows sharded, bit-packed features
        rec = newton_cg(LogisticTask(big), 2, 10, b, fused=fused)
        res[f"full_c3_{int(fused)}_obj"], res[f"full_c3_{int(fused)}_w"] = rec.objectives, rec.final_iterate
    del big
    from paper_2404_11631_b200.sharding import PeerMailbox
    res["nv_peer_used"] = np.array([PeerMailbox.get(sh) is not None])
    np.savez(os.path.join(out, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
