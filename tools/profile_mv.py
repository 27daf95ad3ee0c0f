import sys, torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p
b = p.make_backend("cuda")
a = torch.randn(10_000, 1000, dtype=torch.float64, device="cuda")
q = torch.randn(10_000, dtype=torch.float64, device="cuda")
w = torch.randn(1000, dtype=torch.float64, device="cuda")
for _ in range(3):
    b.matvec_t_device(a, q); b.matvec_device(a, w)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
b.matvec_t_device(a, q); b.matvec_device(a, w)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
