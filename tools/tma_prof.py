import sys; sys.path.insert(0, ".")
import torch
import paper_2404_11631_b200 as p
from paper_2404_11631_b200.newton import logistic_hessian_device
from paper_2404_11631_b200.sampling import synth_classification
data = synth_classification(8192, p.RngStream(42, 0), n_rows=125_000, packed=True)
dw = torch.rand(125_000, dtype=torch.float64, device="cuda") * 0.25
H = torch.empty(8192, 8192, dtype=torch.float64, device="cuda")
logistic_hessian_device(data, dw, out=H, method="tma")
torch.cuda.synchronize()
logistic_hessian_device(data, dw, out=H, method="tma")
torch.cuda.synchronize()
