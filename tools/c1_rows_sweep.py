"""C1 persistent epoch: per-step device time (trace stamps) vs the number of rows N at d=1000 -- how much of a step is the pass and how much the barriers/fold/tail."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
from paper_2404_11631_b200.instances import gen_meanvar_instance
from paper_2404_11631_b200.tasks import MeanVarProblem
d, M = 1000, 25
b = p.make_backend("cuda")
for n in (200, 2000, 10_000):
    prob = MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=True)
    fw_run(prob, FwConfig(3, M, n, p.RngStream(42, 2)), b)
    torch.cuda.synchronize()
    rec = fw_run(prob, FwConfig(10, M, n, p.RngStream(42, 2)), b)
    ns = np.asarray(rec.elapsed_ns, dtype=np.float64)
    st = np.diff(ns)
    within = np.concatenate([st[k*M:(k+1)*M-1] for k in range(1, 9)])
    ends = ns[M - 1::M]
    print(f"N={n}: step (within epoch) median {np.median(within)/1e3:.2f} us, epoch {np.median(np.diff(ends))/1e6:.3f} ms")
