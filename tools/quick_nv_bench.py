"""Quick timing of the newsvendor C2 workload (d=1e4, S=1e5, M=25)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
from paper_2404_11631_b200.instances import gen_newsvendor_instance
from paper_2404_11631_b200.tasks import NewsvendorProblem

d, S, M = 10_000, 100_000, 25
b = p.make_backend("cuda")
task = gen_newsvendor_instance(d, p.RngStream(42, 0))
prob = NewsvendorProblem(task, b)
s = p.RngStream(42, 2)
# resample alone
prob.resample(s, S); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); prob.resample(s, S); e1.record(); e1.synchronize()
print(f"resample d={d} S={S}: {e0.elapsed_time(e1):.3f} ms")
for K in (1, 4):
    torch.cuda.synchronize(); t = time.perf_counter()
    rec = fw_run(prob, FwConfig(K, M, S, p.RngStream(42, 2)), b)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"fw_run K={K} M={M}: {dt*1e3:.1f} ms wall -> {K*M/dt:.1f} it/s; device span {(rec.elapsed_ns[-1])/1e6:.2f} ms; obj[-1]={rec.objectives[-1]:.6f}")
