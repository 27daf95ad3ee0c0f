"""Interleaved A/B of step-kernel configurations (SIMOPT_NV_ITER=W,B,VB) on the pipelined
C2 epoch: each repetition runs every configuration for `epochs` epochs in the same process,
so box-to-box and drift effects cancel.  Prints the median pipelined epoch per config.

  python tools/nv_iter_ab.py "8,3,8 4,3,4 4,7,4/4" [reps] [epochs]   (/4: resample at 40 registers)
env: AB_EPOCHS (overrides epochs), AB_GRAPH=1 (graph engine), AB_TIME_RESAMPLE=1 (resample
events as bench.py records them), AB_CLOCKS=1 (bench.py's NVML sampler running beside).
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.instances import gen_newsvendor_instance  # noqa: E402
from paper_2404_11631_b200.tasks import NewsvendorProblem, make_nv_engine  # noqa: E402

cfgs = sys.argv[1].split() if len(sys.argv) > 1 else ["8,3,8", "4,3,4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
K = int(sys.argv[3]) if len(sys.argv) > 3 else 12
d, S, M = int(os.environ.get("AB_D", 10_000)), 100_000, 25
b = p.make_backend("cuda")
task = gen_newsvendor_instance(d, p.RngStream(42, 0))


TIME_RES = os.environ.get("AB_TIME_RESAMPLE") == "1"
GRAPH = os.environ.get("AB_GRAPH") == "1"
NOSIDE = os.environ.get("AB_NOSIDE") == "1"
TRACE = os.environ.get("AB_TRACE") == "1"
if TRACE:  # every engine event timed
    _Ev = torch.cuda.Event
    torch.cuda.Event = lambda enable_timing=False, **kw: _Ev(enable_timing=True, **kw)  # CUDA-graph epochs (NvFwGraphEngine)
K = int(os.environ.get("AB_EPOCHS", K))


def run():
    prob = NewsvendorProblem(task, b)
    eng = make_nv_engine(prob, M, K, b.chunk_size, graph=GRAPH)
    if NOSIDE:  # diagnostic: drop the per-step recording kernels (records become garbage)
        real = eng.lib

        class _Lib:
            def __getattr__(self, n):
                if n in ("simopt_nv_cost_terms", "simopt_tree_sums2", "simopt_timestamp"):
                    return lambda *a_: 0
                return getattr(real, n)
        eng.lib = _Lib()
    st = p.RngStream(42, 2)
    eng.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    for k in range(K):
        if k == 2:
            torch.cuda.synchronize()
            t0.record()
        eng.enqueue_epoch(k, st, S, time_resample=TIME_RES, next_samples=S if k + 1 < K else None)
    eng.finish()
    t1.record()
    torch.cuda.synchronize()
    if TRACE:  # per-epoch spacing of the step-sequence ends
        ends = [eng.steps_done[k] for k in range(K)]
        print("epoch spacing ms:", " ".join(f"{ends[k - 1].elapsed_time(ends[k]):.2f}" for k in range(1, K)))
    return t0.elapsed_time(t1) / (K - 2)


if os.environ.get("AB_CLOCKS") == "1":  # bench.py's NVML clock sampler running beside
    import bench
    clk = bench.ClockSampler(torch.cuda.current_device())
    clk.__enter__()
res = {c: [] for c in cfgs}
run()  # warm-up
for r in range(reps):
    for c in cfgs:
        it, _, rc = c.partition("/")  # "W,B,V[,P]/R": R = the resample's register cap (3: 48 registers, 4: 40; default by shard size)
        os.environ["SIMOPT_NV_ITER"] = it
        if rc:
            os.environ["SIMOPT_NV_WS_REGCAP"] = rc
        else:
            os.environ.pop("SIMOPT_NV_WS_REGCAP", None)
        res[c].append(run())
for c in cfgs:
    v = res[c]
    print(f"{c:10s} epoch median {statistics.median(v):.3f} ms  min {min(v):.3f}  "
          f"-> {M / statistics.median(v) * 1e3:.0f} FW it/s   ({', '.join(f'{x:.3f}' for x in v)})")
