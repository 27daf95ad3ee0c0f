"""BASELINE.json configs[4] at full size on ONE B200: logistic Newton with the explicit
X^T D X Hessian, d = 8192, N = 10^7 (bit-packed features: 10.2 GB; fp64 would be 655 GB).
Times one Newton iteration (Hessian on the FP64 tensor pipe + fused gradient + CG solve)
with CUDA events.  Per-GPU work at 8 GPUs is 1/8 of the Hessian plus one 537 MB allreduce.

  python tools/c5_full.py [N]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.newton import logistic_hessian_device, newton_explicit  # noqa: E402
from paper_2404_11631_b200.sampling import synth_classification  # noqa: E402
from paper_2404_11631_b200.tasks import LogisticTask  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
d = 8192
t0 = time.perf_counter()
data = synth_classification(d, p.RngStream(42, 0), n_rows=N, packed=True)
torch.cuda.synchronize()
t_inst = time.perf_counter() - t0
b = p.make_backend("cuda")
dw = torch.rand(N, dtype=torch.float64, device="cuda") * 0.25
H = torch.empty(d, d, dtype=torch.float64, device="cuda")
logistic_hessian_device(data, dw, out=H)  # warm
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
logistic_hessian_device(data, dw, out=H)
e1.record()
e1.synchronize()
h_ms = e0.elapsed_time(e1)
e0.record()
rec = newton_explicit(LogisticTask(data), 1, 20, b)
e1.record()
e1.synchronize()
it_ms = e0.elapsed_time(e1)
flops = N * d * (d + 1)  # SYRK convention
print(json.dumps({"config": "C5 logistic explicit-Hessian Newton d=8192 N=1e7 (full, 1 GPU, bit-packed)",
                  "N": N, "d": d, "instance_s": t_inst, "hessian_ms": h_ms,
                  "hessian_tflops_syrk_convention": flops / (h_ms / 1e3) / 1e12,
                  "newton_iteration_ms": it_ms, "newton_iterations_per_s": 1e3 / it_ms,
                  "objective": rec.final_objective}), flush=True)
