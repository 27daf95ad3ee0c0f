"""C1's per-epoch draw, part by part (CUDA events): the exact affine normals of X (N x d),
the exact-tree column sums for the mean, and the scale-subtract."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200 import _lib  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402
from paper_2404_11631_b200.tasks import MeanVarProblem  # noqa: E402

d, n = 1000, 10_000
b = p.make_backend("cuda")
prob = MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=True)
st = p.RngStream(42, 2)
prob.resample_slot(st, n, 0)
torch.cuda.synchronize()
x, mean, ones = prob._slots[0]


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


mu, sd = prob._mu_dev, prob._sd_dev
t_draw = timed(lambda: _lib.call("simopt_sample_returns_diag", _lib.stream_ptr(), *st.words(), n, d,
                                 _lib.ptr(mu), _lib.ptr(sd), _lib.ptr(x)))
t_cols = timed(lambda: b.matvec_t_device(x, ones))
t_slot = timed(lambda: prob.resample_slot(st, n, 0))
print(f"C1 draw parts (us): normals {t_draw:.1f}, exact column sums {t_cols:.1f}, whole resample_slot {t_slot:.1f}")
