"""Golden trajectories at BASELINE.json sizes, from the REAL reference (sobench).

Runs only in the build container, where /root/reference exists (about 4 minutes
on 8 vCPU, ~30 GB of host memory):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/gen_full.py [c2] [c3] [c4]

Writes tests/golden/full_*.npz (trajectories only: objectives per step, final
iterate).  tests/test_gpu_full_size.py runs the CUDA path on the same inputs
and compares: exact modes bit for bit, fused modes within the north star's 1e-8.

* full_c2: BASELINE configs[1] -- sobench fw_run of NewsvendorProblem, d=10^4,
  S=10^5, M=25, 3 epochs (bench.py's instance and optimizer streams), sobench
  ParallelBackend (bitwise equal to SequentialBackend by the reference's contract,
  tests/test_backend.py).
* full_c3: BASELINE configs[2] -- Newton-CG on the N-generalised classification
  instance (d=10^3, N=10^6; oracle.synth_classification, pinned to the reference's
  synth_classification at N=30d), with the reference's own logistic_gradient,
  logistic_hvp, logistic_loss and fixed-tree dot in oracle.newton_cg's recurrence.
* full_c4: BASELINE configs[3]'s d (2*10^4) at N = 2*10^4 scenarios -- sobench fw_run
  of MeanVarProblem, one epoch of M=25 (the reference cannot hold C4's 160 GB X).
"""
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from sobench import _kernels  # noqa: E402
from sobench.backend import make_backend  # noqa: E402
from sobench.bench import gen_meanvar_instance, gen_newsvendor_instance  # noqa: E402
from sobench.frank_wolfe import FwConfig, fw_run  # noqa: E402
from sobench.sampling import ClassificationData, RngStream  # noqa: E402
from sobench.tasks import (MeanVarProblem, NewsvendorProblem, logistic_gradient,  # noqa: E402
                           logistic_hvp, logistic_loss)

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    print("wrote", name, {k: np.asarray(v).shape for k, v in arrays.items()}, flush=True)


def c2(b):
    d, S, M, K = 10_000, 100_000, 25, 3
    task = gen_newsvendor_instance(d, RngStream(42, 0))
    rec = fw_run(NewsvendorProblem(task, b), FwConfig(K, M, S, RngStream(42, 2)), b)
    save("full_c2", objectives=rec.objectives, final_iterate=rec.final_iterate,
         meta=np.array([d, S, M, K]))


def newton_cg_ref(x, z, iterations, cg_iters, b):
    """oracle.newton_cg's recurrence (oracle/oracle.py) over the reference's functions."""
    data = ClassificationData(features=x, labels=z, true_weights=np.zeros(x.shape[1]))
    n = x.shape[1]
    w = np.zeros(n)
    objs = []
    for _ in range(iterations):
        g = logistic_gradient(w, data, None, b)
        p = np.zeros(n)
        r = -1.0 * g
        dd = r.copy()
        rr = b.dot(r, r)
        for _ in range(cg_iters):
            if rr == 0.0:
                break
            hd = logistic_hvp(w, dd, data, None, b)
            alpha = rr / b.dot(dd, hd)
            p = p + alpha * dd
            r = r - alpha * hd
            rr_new = b.dot(r, r)
            beta = rr_new / rr
            dd = r + beta * dd
            rr = rr_new
        w = w + p
        objs.append(logistic_loss(w, data, None, b))
    return np.array(objs), w


def c3(b):
    from oracle import oracle as orc
    # the recurrence over sobench == oracle.newton_cg, checked on a small instance first
    xs, zs, _ = orc.synth_classification(40, orc.Stream(42, 0), n_rows=5000)
    o1, w1 = orc.newton_cg(xs, zs, iterations=2, cg_iters=6)
    o2, w2 = newton_cg_ref(xs, zs, 2, 6, b)
    assert np.array_equal(o1, o2) and np.array_equal(w1, w2)
    d, N, iters, kcg = 1_000, 1_000_000, 2, 10
    t = time.time()
    x, z, w_true = orc.synth_classification(d, orc.Stream(42, 0), n_rows=N)
    print(f"c3 instance {time.time() - t:.1f} s", flush=True)
    objs, w = newton_cg_ref(x, z, iters, kcg, b)
    save("full_c3", objectives=objs, final_iterate=w, labels_sum=np.array([z.sum()]),
         w_true=w_true, meta=np.array([d, N, iters, kcg]))


def c4(b):
    d, N, M, K = 20_000, 20_000, 25, 1
    task = gen_meanvar_instance(d, RngStream(42, 0))
    rec = fw_run(MeanVarProblem(task, b), FwConfig(K, M, N, RngStream(42, 2)), b)
    save("full_c4", objectives=rec.objectives, final_iterate=rec.final_iterate,
         meta=np.array([d, N, M, K]))


if __name__ == "__main__":
    _kernels.warmup()
    b = make_backend("parallel", workers=os.cpu_count())
    which = sys.argv[1:] or ["c2", "c3", "c4"]
    for name in which:
        t = time.time()
        globals()[name](b)
        print(f"{name}: {time.time() - t:.1f} s", flush=True)
