"""C1 fused FW run: device time per epoch (from the trace's %globaltimer stamps) against
the wall clock of the host loop, to see whether the host or the device bounds the epoch.

  python tools/c1_timeline.py [epochs]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402
from paper_2404_11631_b200.tasks import MeanVarProblem  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
d, n, M = 1000, 10_000, 25
b = p.make_backend("cuda")
prob = MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=True)
fw_run(prob, FwConfig(3, M, n, p.RngStream(42, 2)), b)
torch.cuda.synchronize()
t = time.perf_counter()
rec = fw_run(prob, FwConfig(K, M, n, p.RngStream(42, 2)), b)
torch.cuda.synchronize()
wall = (time.perf_counter() - t) * 1e3
ns = np.asarray(rec.elapsed_ns, dtype=np.float64)
ends = ns[M - 1::M]  # stamp of each epoch's last step
ep = np.diff(ends) / 1e6
steps = np.array([(ns[k * M + M - 1] - ns[k * M]) / 1e6 for k in range(K)])
print(f"{K} epochs: wall {wall:.2f} ms ({wall / K:.3f} ms/epoch); device epoch spacing median "
      f"{np.median(ep):.3f} ms; steps 1..M of an epoch median {np.median(steps):.3f} ms "
      f"({np.median(steps) / (M - 1) * 1e3:.1f} us per step)")
