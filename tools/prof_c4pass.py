"""One fused mean-variance pass at the C4 per-GPU slice (N = 1.25e5, d = 2e4) for ncu."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.fused import MV, fused_rows  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402
from paper_2404_11631_b200.tasks import MeanVarProblem  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
b = p.make_backend("cuda")
prob = MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=True)
prob.resample(p.RngStream(42, 2), N)
ss = prob.sample_set
w = torch.full((d,), 1.0 / d, dtype=torch.float64, device="cuda")
g = torch.empty(d, dtype=torch.float64, device="cuda")
q = torch.empty(1, dtype=torch.float64, device="cuda")
for _ in range(3):
    fused_rows(MV, ss.samples, w, center=ss.mean, col_scale=1.0 / (N - 1), col_out=g, scalar_out=q)
torch.cuda.synchronize()
