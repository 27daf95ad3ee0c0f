import sys, torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p
n = 500_000_000
out = torch.empty(n, dtype=torch.float64, device="cuda")
p.standard_normal_device(p.RngStream(1, 2), n, out); torch.cuda.synchronize()
p.standard_normal_device(p.RngStream(1, 3), n, out); torch.cuda.synchronize()
