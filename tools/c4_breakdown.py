"""Where the C4 epoch goes on one GPU (full size by default): the draw of X (exact glibc
normals, affine), the exact column sums for the mean, and the M+1 fused passes, each timed
alone with CUDA events.

  python tools/c4_breakdown.py [N] [d]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.fused import MV, fused_rows  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402
from paper_2404_11631_b200.tasks import MeanVarProblem  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
b = p.make_backend("cuda")
prob = MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=True)


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


st = p.RngStream(42, 2)
t_all = timed(lambda: prob.resample(st, N))
ss = prob.sample_set
x, mean = ss.samples, ss.mean
ones = torch.ones(N, dtype=torch.float64, device="cuda")
t_mean = timed(lambda: b.matvec_t_device(x, ones))
w = torch.full((d,), 1.0 / d, dtype=torch.float64, device="cuda")
g = torch.empty(d, dtype=torch.float64, device="cuda")
q = torch.empty(1, dtype=torch.float64, device="cuda")
t_pass = timed(lambda: fused_rows(MV, x, w, center=mean, col_scale=1.0 / (N - 1), col_out=g,
                                  scalar_out=q))
gb = 8 * N * d / 1e9
from paper_2404_11631_b200.fused import fused_geometry  # noqa: E402
print("pass geometry:", fused_geometry(MV, d))
print(f"N={N} d={d} ({gb:.1f} GB): resample (draw + exact mean) {t_all:.1f} ms, of which the exact "
      f"column sums {t_mean:.1f} ms ({gb / t_mean:.2f} TB/s); fused pass {t_pass:.1f} ms "
      f"({gb / t_pass:.2f} TB/s); epoch estimate {t_all + 26 * t_pass:.0f} ms")
