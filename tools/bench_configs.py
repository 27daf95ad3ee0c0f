"""Throughput of every BASELINE.json config on one B200 (secondary to bench.py's headline).

Prints one JSON line per config.  Per-GPU slices are used where the full
config is multi-GPU or exceeds one GPU's HBM (stated in each line).
CUDA events on the launching stream; >= 3 warm-up steps; inputs > L2 except C1.

  python tools/bench_configs.py [c1 c3 c4 c5 xtdx]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2404_11631_b200 as p  # noqa: E402
from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run  # noqa: E402
from paper_2404_11631_b200.instances import gen_meanvar_instance  # noqa: E402
from paper_2404_11631_b200.tasks import LogisticTask, MeanVarProblem  # noqa: E402


def timed(fn, warm=3, reps=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def meanvar(tag, d, n, M=25, epochs=8, fused=False):
    b = p.make_backend("cuda")
    prob = MeanVarProblem(gen_meanvar_instance(d, p.RngStream(42, 0)), b, fused=fused)
    s = p.RngStream(42, 2)
    ms = timed(lambda: fw_run(prob, FwConfig(epochs, M, n, s), b), warm=1, reps=2)
    it_s = epochs * M / (ms / 1e3)
    # algorithmic bytes per iteration: one read of X + the amortized
    # per-epoch resample write/colsum read, 8 N d (1 + 1/M)
    alg = 8 * n * d * (1 + 1 / M)
    print(json.dumps({"config": tag, "d": d, "N": n, "M": M, "fused": fused,
                      "fw_iterations_per_s": it_s, "ms_per_epoch": ms / epochs,
                      "passes_per_iteration": (M + 1) / M if fused else (2 * M + 1) / M,
                      "algorithmic_GBps": alg * it_s / 1e9}), flush=True)


def newton(tag, d, n, k_cg=10, iters=2, fused=True, packed=False):
    from paper_2404_11631_b200.newton import newton_cg
    from paper_2404_11631_b200.sampling import synth_classification
    b = p.make_backend("cuda")
    task = LogisticTask(synth_classification(d, p.RngStream(42, 0), n_rows=n, packed=packed))
    ms = timed(lambda: newton_cg(task, iters, k_cg, b, fused=fused), warm=1, reps=2)
    it_s = iters / (ms / 1e3)
    passes = k_cg + 1 if fused else 2 * k_cg + 2
    alg = 8 * n * d * (k_cg + 1)  # one read of X per gradient / HVP
    print(json.dumps({"config": tag, "d": d, "N": n, "k_cg": k_cg, "fused": fused, "packed": packed,
                      "newton_iterations_per_s": it_s,
                      "ms_per_iteration": ms / iters, "passes_over_X": passes,
                      "achieved_GBps": passes * 8 * n * d * it_s / 1e9,
                      "algorithmic_GBps": alg * it_s / 1e9}), flush=True)


def sqn(tag, d, n, iters=2000, packed=False, graph=True):
    """The reference's own classification solver (sqn.py) at C3 scale, bench.py:57-74
    parameters (L=10, M=25, beta=2, b=50, b_H=300); exact trees, bit-exact traces.
    Per iteration: one full-data loss pass over X (sqn.py:171) dominates.  K = 2000, the
    reference's classification default (bench.py:89)."""
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.sqn import SqnConfig, sqn_run
    b = p.make_backend("cuda")
    task = LogisticTask(synth_classification(d, p.RngStream(42, 0), n_rows=n, packed=packed))

    def run():
        cfg = SqnConfig(pair_every=10, memory=25, beta=2.0, grad_batch=50, hess_batch=300,
                        iterations=iters, stream=p.RngStream(42, 2))
        sqn_run(task, cfg, b, graph=graph)
    ms = timed(run, warm=1, reps=1)
    it_s = iters / (ms / 1e3)
    x_bytes = n * d / 8 if packed else 8 * n * d
    print(json.dumps({"config": tag, "d": d, "N": n, "packed": packed, "graph": graph,
                      "iterations": iters,
                      "sqn_iterations_per_s": it_s, "ms_per_iteration": ms / iters,
                      "loss_pass_GBps": x_bytes * it_s / 1e9}), flush=True)


def xtdx(tag, d, n, packed=False, method="dmma"):
    from paper_2404_11631_b200.newton import logistic_hessian_device
    from paper_2404_11631_b200.sampling import synth_classification
    data = synth_classification(d, p.RngStream(42, 0), n_rows=n, packed=packed)
    dw = torch.rand(n, dtype=torch.float64, device="cuda") * 0.25
    H = torch.empty(d, d, dtype=torch.float64, device="cuda")
    ms = timed(lambda: logistic_hessian_device(data, dw, out=H, method=method), warm=1, reps=3)
    flops_syrk = n * d * (d + 1)  # SYRK convention
    print(json.dumps({"config": tag, "d": d, "N": n, "ms": ms,
                      "tflops_syrk_convention": flops_syrk / (ms / 1e3) / 1e12,
                      "note": "upper-triangle tiles computed, mirrored"}), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c3", "c4", "xtdx"]
    if "c1" in which:
        meanvar("C1 meanvar d=1e3 N=1e4 (exact tree)", 1000, 10_000)
        meanvar("C1 meanvar d=1e3 N=1e4 (fused)", 1000, 10_000, fused=True)
    if "c4" in which:
        meanvar("C4 meanvar d=2e4, per-GPU slice N=1.25e5 of N=1e6 on 8 GPUs (exact tree)",
                20_000, 125_000, epochs=2)
        meanvar("C4 meanvar d=2e4, per-GPU slice N=1.25e5 of N=1e6 on 8 GPUs (fused)",
                20_000, 125_000, epochs=2, fused=True)
    if "c3" in which:
        newton("C3 logistic Newton-CG d=1e3 N=1e6 (exact tree)", 1000, 1_000_000, fused=False)
        newton("C3 logistic Newton-CG d=1e3 N=1e6 (fused)", 1000, 1_000_000)
        newton("C3 logistic Newton-CG d=1e3 N=1e6 (fused, bit-packed features)", 1000, 1_000_000,
               packed=True)
    if "sqn" in which:
        sqn("C3-scale SQN (reference solver) d=1e3 N=1e6", 1000, 1_000_000)
        sqn("C3-scale SQN (reference solver) d=1e3 N=1e6 (bit-packed features)", 1000, 1_000_000,
            packed=True)
        sqn("C3-scale SQN (reference solver) d=1e3 N=1e6 (bit-packed, eager iteration)", 1000,
            1_000_000, packed=True, graph=False)
    if "tma" in which:
        xtdx("C5 X^T D X slice (tc)", 8192, 125_000, packed=True, method="tc")
        xtdx("C5 X^T D X slice (tma)", 8192, 125_000, packed=True, method="tma")
    if "sqn_ab" in which:  # graph vs eager, alternating
        for g in (True, False, True, False):
            sqn(f"SQN packed ab graph={g}", 1000, 1_000_000, packed=True, graph=g)
    if "sqn_small" in which:  # the reference's own sizes: N = 30 d (sampling.py:241)
        for d in (100, 1000):
            for g in (True, False):
                sqn(f"SQN d={d} N=30d (reference bench size), {'graph' if g else 'eager'}", d, 30 * d,
                    graph=g)
    if "xtdx" in which:
        xtdx("C5 X^T D X d=8192, per-GPU slice N=1.25e5 (fp64 X)", 8192, 125_000)
        xtdx("C5 X^T D X d=8192, per-GPU slice N=1.25e5 (bit-packed X, DMMA)", 8192, 125_000,
             packed=True)
        xtdx("C5 X^T D X d=8192, per-GPU slice N=1.25e5 (bit-packed X, u8 IMMA limbs)", 8192,
             125_000, packed=True, method="i8")
        xtdx("C5 X^T D X d=8192, per-GPU slice N=1.25e5 (bit-packed X, tcgen05 i8 limbs, TMEM)", 8192,
             125_000, packed=True, method="tc")
        xtdx("C5 X^T D X d=8192, per-GPU slice N=1.25e5 (bit-packed X, tcgen05 i8 limbs, TMA operands)",
             8192, 125_000, packed=True, method="tma")
