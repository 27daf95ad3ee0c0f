"""One warm-up + one profiled newsvendor epoch at C2 size (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
from paper_2404_11631_b200.instances import gen_newsvendor_instance
from paper_2404_11631_b200.tasks import NewsvendorProblem

d = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
b = p.make_backend("cuda")
prob = NewsvendorProblem(gen_newsvendor_instance(d, p.RngStream(42, 0)), b)
fw_run(prob, FwConfig(1, 25, S, p.RngStream(42, 2)), b)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fw_run(prob, FwConfig(1, 25, S, p.RngStream(42, 3)), b)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
