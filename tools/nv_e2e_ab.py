"""Where the C2 end-to-end time goes: fw_run (60 epochs, host instance arrays) with the
eager engine vs the CUDA-graph engine, the host's per-epoch enqueue cost, and the
caching allocator's device allocations / retries during each run.

  python tools/nv_e2e_ab.py [d] [S] [epochs]
"""
import gc
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200 import tasks  # noqa: E402
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run  # noqa: E402
from paper_2404_11631_b200.instances import gen_newsvendor_instance  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
E = int(sys.argv[3]) if len(sys.argv) > 3 else 60
M = 25
b = p.make_backend("cuda")
task = gen_newsvendor_instance(d, p.RngStream(42, 0))
orig = tasks.make_nv_engine
enq_times = []


def forced(graph):
    def make(prob, inner, epochs, chunk, graph_=None):
        eng = orig(prob, inner, epochs, chunk, graph=graph)
        f = eng.enqueue_epoch

        def timed(*a, **k):
            t = time.perf_counter()
            r = f(*a, **k)
            enq_times.append(time.perf_counter() - t)
            return r
        eng.enqueue_epoch = timed
        return eng
    return make


def stats():
    s = torch.cuda.memory_stats()
    return s.get("num_device_alloc", 0), s.get("num_device_free", 0), s.get("num_alloc_retries", 0)


for graph in [False, True] * 3:
    tasks.make_nv_engine = forced(graph)
    fw_run(tasks.NewsvendorProblem(task, b), FwConfig(3, M, S, p.RngStream(42, 2)), b)
    torch.cuda.synchronize()
    enq_times.clear()
    s0 = stats()
    t = time.perf_counter()
    rec = fw_run(tasks.NewsvendorProblem(task, b), FwConfig(E, M, S, p.RngStream(42, 2)), b)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    s1 = stats()
    et = sorted(enq_times)
    slow = [i for i, x in enumerate(enq_times) if x > 5e-3]
    print(f"graph={graph}: {E} epochs {dt * 1e3:.1f} ms = {E * M / dt:.0f} FW it/s; "
          f"enqueue per epoch median {et[len(et) // 2] * 1e3:.2f} ms max {et[-1] * 1e3:.2f} ms "
          f"(slow epochs {slow}); device alloc/free/retries during run "
          f"{[b_ - a_ for a_, b_ in zip(s0, s1)]}; reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB; "
          f"final objective {rec.objectives[-1]!r}", flush=True)
    gc.collect()
