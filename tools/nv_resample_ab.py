"""A/B of the newsvendor resample kernels: layouts equal (off exactly, keys as per-bucket
multisets) and the time of each variant (CUDA events, C2 size by default).

  python tools/nv_resample_ab.py [d] [S] [VAR=v,v,... ...]

Each extra argument names an environment variable and the values to try, e.g.
SIMOPT_NV_PHX=0,1 (the launcher reads these per call).
"""
import itertools
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.instances import gen_newsvendor_instance  # noqa: E402
from paper_2404_11631_b200.tasks import NewsvendorProblem  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
grid = [a.split("=", 1) for a in sys.argv[1:] if "=" in a]
d = int(args[0]) if len(args) > 0 else 10_000
S = int(args[1]) if len(args) > 1 else 100_000
b = p.make_backend("cuda")
prob = NewsvendorProblem(gen_newsvendor_instance(d, p.RngStream(42, 0)), b)


def run(reps=7):
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
    return sorted(ts)[len(ts) // 2], prob.dev.keys.clone(), prob.dev.off.clone()


def canon(keys):
    """Per-segment sorted keys (order inside a bucket is free)."""
    k = keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    rows = k.view(d, S)
    return torch.cat([torch.sort(rows[:, s0:s0 + 4096], dim=1).values for s0 in range(0, S, 4096)], 1)


ref = None
names = [g[0] for g in grid]
for combo in itertools.product(*[g[1].split(",") for g in grid]) if grid else [()]:
    for n, v in zip(names, combo):
        os.environ[n] = v
    t, k, o = run()
    ck = canon(k)
    if ref is None:
        ref = (ck, o)
        same = True
    else:
        same = torch.equal(o, ref[1]) and torch.equal(ck, ref[0])
        del ck
    print(f"{dict(zip(names, combo))}: median {t:.3f} ms  layout equal to first: {same}", flush=True)
