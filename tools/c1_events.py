"""C1 fused FW run with timed events around each epoch's draw (generator stream) and steps
(main stream): prints the device timeline of a few epochs (ms from the first event)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200 import tasks  # noqa: E402
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402

marks = []


def mark(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks.append((name, e))


orig_slot = tasks.MeanVarProblem.resample_slot
orig_run = tasks.MvFwEngine.run_epoch


def slot(self, stream, n, s):
    mark(f"draw{s}+")
    r = orig_slot(self, stream, n, s)
    mark(f"draw{s}-")
    return r


def run(self, k, n):
    mark(f"ep{k}+")
    r = orig_run(self, k, n)
    mark(f"ep{k}-")
    return r


tasks.MeanVarProblem.resample_slot = slot
tasks.MvFwEngine.run_epoch = run
d, n, M = 1000, 10_000, 25
b = p.make_backend("cuda")
prob = tasks.MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=True)
fw_run(prob, FwConfig(3, M, n, p.RngStream(42, 2)), b)
torch.cuda.synchronize()
marks.clear()
fw_run(prob, FwConfig(8, M, n, p.RngStream(42, 2)), b)
torch.cuda.synchronize()
t0 = marks[0][1]
print("  ".join(f"{nm}@{t0.elapsed_time(e):.3f}" for nm, e in marks))
