"""Profiled fused passes (for ncu): C3 Newton-CG iteration (d=1e3, N=1e6) and a C4
per-GPU-slice mean-variance fused FW epoch (d=2e4, N=1.25e5).

  python tools/profile_fused.py [c3|c3bits|c4]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402
from paper_2404_11631_b200.newton import newton_cg  # noqa: E402
from paper_2404_11631_b200.sampling import synth_classification  # noqa: E402
from paper_2404_11631_b200.tasks import LogisticTask, MeanVarProblem  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
b = p.make_backend("cuda")
if which in ("c3", "c3bits"):
    task = LogisticTask(synth_classification(1000, p.RngStream(42, 0), n_rows=1_000_000,
                                             packed=which == "c3bits"))
    run = lambda: newton_cg(task, 1, 10, b)  # noqa: E731
else:
    prob = MeanVarProblem(gen_meanvar_instance(20_000, p.RngStream(42, 0)), b, fused=True)
    run = lambda: fw_run(prob, FwConfig(1, 25, 125_000, p.RngStream(42, 2)), b)  # noqa: E731
run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
