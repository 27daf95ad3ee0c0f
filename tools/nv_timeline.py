"""Per-epoch timeline of the pipelined C2 loop (eager engine): when each epoch's resample,
step sequence and records start and end, relative to a common origin (CUDA events on the
streams that run them).  Shows where the steady-state epoch spacing goes beyond the
resample's own duration.

  python tools/nv_timeline.py [d] [epochs]
"""
import sys

import torch

sys.path.insert(0, ".")
_Ev = torch.cuda.Event
torch.cuda.Event = lambda enable_timing=False, **kw: _Ev(enable_timing=True, **kw)
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.instances import gen_newsvendor_instance  # noqa: E402
from paper_2404_11631_b200.tasks import NewsvendorProblem, NvFwEngine  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
S, M = 100_000, 25
b = p.make_backend("cuda")
task = gen_newsvendor_instance(d, p.RngStream(42, 0))


class Timed(NvFwEngine):
    def _enqueue_steps(self, k, sp, ssp):
        e = torch.cuda.Event()
        e.record(self.hi)
        self.step_start[k] = e
        super()._enqueue_steps(k, sp, ssp)


for rep in range(2):
    prob = NewsvendorProblem(task, b)
    eng = Timed(prob, M, K, b.chunk_size)
    eng.step_start = {}
    st = p.RngStream(42, 2)
    torch.cuda.synchronize()
    org = torch.cuda.Event()
    org.record()
    eng.start()
    for k in range(K):
        eng.enqueue_epoch(k, st, S, time_resample=True, next_samples=S if k + 1 < K else None)
    eng.finish()
    torch.cuda.synchronize()
    if rep == 0:
        continue
    t = org.elapsed_time
    print(" k | resample start..end (dur) | steps start..end (dur) | records end")
    for k in range(K):
        r0, r1 = eng.resample_events[k]
        print(f"{k:2d} | {t(r0):8.3f}..{t(r1):8.3f} ({r0.elapsed_time(r1):.3f}) | "
              f"{t(eng.step_start[k]):8.3f}..{t(eng.steps_done[k]):8.3f} "
              f"({eng.step_start[k].elapsed_time(eng.steps_done[k]):.3f}) | {t(eng.epoch_done[k]):8.3f}")
