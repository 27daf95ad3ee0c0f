"""One warm-up + one profiled mean-variance FW epoch (for ncu): C1 by default.

  python tools/profile_mv.py [d] [N] [fused 0|1]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402
from paper_2404_11631_b200.tasks import MeanVarProblem  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000
fused = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
b = p.make_backend("cuda")
prob = MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=fused)
fw_run(prob, FwConfig(2, 25, n, p.RngStream(42, 2)), b)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fw_run(prob, FwConfig(1, 25, n, p.RngStream(42, 3)), b)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
