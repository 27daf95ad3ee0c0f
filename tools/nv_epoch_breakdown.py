"""Where the C2 epoch goes: resample alone, the 26 step kernels alone, and the pipelined
epoch (next resample overlapping this epoch's steps), CUDA events per stream.

  python tools/nv_epoch_breakdown.py [d] [S] [epochs]
"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.instances import gen_newsvendor_instance  # noqa: E402
from paper_2404_11631_b200.tasks import NewsvendorProblem, NvFwEngine  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
K = int(sys.argv[3]) if len(sys.argv) > 3 else 12
M = 25
b = p.make_backend("cuda")
task = gen_newsvendor_instance(d, p.RngStream(42, 0))


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


class Timed(NvFwEngine):
    def _enqueue_steps(self, k, sp, ssp):
        self.step_ev.setdefault(k, [None, None])[0] = ev()
        super()._enqueue_steps(k, sp, ssp)
        self.step_ev[k][1] = ev()


def run(pipelined):
    prob = NewsvendorProblem(task, b)
    eng = Timed(prob, M, K, b.chunk_size)
    eng.step_ev = {}
    st = p.RngStream(42, 2)
    eng.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    for k in range(K):
        if k == 2:
            torch.cuda.synchronize()
            t0.record()
        nxt = S if (pipelined and k + 1 < K) else None
        eng.enqueue_epoch(k, st, S, time_resample=True, next_samples=nxt)
        if not pipelined:
            eng.finish()
            torch.cuda.synchronize()
    eng.finish()
    t1.record()
    torch.cuda.synchronize()
    res = [a.elapsed_time(b_) for a, b_ in eng.resample_events[2:]]
    steps = [eng.step_ev[k][0].elapsed_time(eng.step_ev[k][1]) for k in range(2, K)]
    print(f"{'pipelined' if pipelined else 'serial   '}: epoch {t0.elapsed_time(t1) / (K - 2):.3f} ms, "
          f"resample {statistics.mean(res):.3f} ms, steps span {statistics.mean(steps):.3f} ms "
          f"(per step {statistics.mean(steps) / (M + 1) * 1e3:.1f} us)")


run(False)
run(True)
