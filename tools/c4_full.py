"""BASELINE.json configs[3] at full size on ONE B200: mean-variance FW, d = 2*10^4 assets,
N = 10^6 scenarios per epoch (fp64 X: 160 GB of the 180 GB HBM), fused single-pass mode.
The 8-GPU configuration shards these rows (20 GB per GPU) with one d+1 allreduce per step.

  python tools/c4_full.py [N] [epochs]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402
from paper_2404_11631_b200.tasks import MeanVarProblem  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2
d, M = 20_000, 25
b = p.make_backend("cuda")
prob = MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=True)
fw_run(prob, FwConfig(1, M, N, p.RngStream(42, 2)), b)  # warm (allocates X once)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
rec = fw_run(prob, FwConfig(K, M, N, p.RngStream(42, 3)), b)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1)
it_s = K * M / (ms / 1e3)
alg = 8 * N * d * (1 + 1 / M)
print(json.dumps({"config": "C4 meanvar d=2e4 N=1e6 (full, 1 GPU, fused)", "N": N, "d": d, "M": M,
                  "epochs": K, "ms_per_epoch": ms / K, "fw_iterations_per_s": it_s,
                  "algorithmic_GBps": alg * it_s / 1e9,
                  "peak_mem_GB": torch.cuda.max_memory_allocated() / 1e9,
                  "final_objective": rec.final_objective}), flush=True)
