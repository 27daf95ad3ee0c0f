"""A/B of the newsvendor resample kernels: layouts equal (off exactly, keys as per-bucket
multisets) and the time of each variant/occupancy (CUDA events, C2 size by default).

  python tools/nv_resample_ab.py [d] [S]
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.instances import gen_newsvendor_instance  # noqa: E402
from paper_2404_11631_b200.tasks import NewsvendorProblem  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
b = p.make_backend("cuda")
prob = NewsvendorProblem(gen_newsvendor_instance(d, p.RngStream(42, 0)), b)


def run(variant, reps=5):
    os.environ["SIMOPT_NV_RESAMPLE"] = str(variant)
    prob.dev.resample(p.RngStream(42, 2), S)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        prob.dev.resample(p.RngStream(42, 2), S)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    keys = prob.dev.keys.clone()
    off = prob.dev.off.clone()
    return min(ts), keys, off


def canon(keys):
    """Per-segment sorted keys (order inside a bucket is free)."""
    k = keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    rows = k.view(d, S)
    out = []
    for s0 in range(0, S, 4096):
        out.append(torch.sort(rows[:, s0:s0 + 4096], dim=1).values)
    return torch.cat(out, dim=1)


t1, k1, o1 = run(1)
print(f"k_nv_resample (single-role, 6 CTAs/SM): {t1:.3f} ms")
t2, k2, o2 = run(0)
same = torch.equal(o1, o2) and torch.equal(canon(k1), canon(k2))
print(f"k_nv_resample_ws (warp-specialised, default): {t2:.3f} ms  layout equal: {same}")
