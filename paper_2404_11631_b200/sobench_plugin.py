"""Register the ``"cuda"`` backend inside the reference package itself.

``install()`` extends an importable ``sobench`` (the reference, e.g. installed into
``baseline/_ref``) so that its own configuration, CLI, CSV traces and summaries run the
B200 path unchanged:

* ``sobench.backend.make_backend("cuda")`` returns this package's ``CudaBackend``
  (the reference's factory raises ConfigurationError for unknown kinds,
  sobench/backend.py:207-213; ``"gpu"`` keeps raising, tests/test_backend.py:214-216);
* ``sobench.bench.run_cell`` (bench.py:152-184) dispatches ``backend_kind == "cuda"`` to
  this package's device-resident problems, instance generators and drivers with the same
  streams (instance ``RngStream(seed, 0)``, repetition ``RngStream(seed, 2 + rep)``), and
  returns a RunRecord with the reference's fields, which ``write_trace_csv`` /
  ``summarize`` consume as they are;
* ``sobench.bench.run_bench`` additionally writes ``kernels.csv`` for the cuda cells: the
  dominant kernels' CUDA-event times with their algorithmic bytes and fraction of the
  measured HBM peak (the per-kernel roofline columns).

    python -m paper_2404_11631_b200.sobench_plugin run --task newsvendor --sizes 1000 \\
        --backend cuda,parallel --reps 3

runs the reference CLI (sobench/cli.py) with the cuda backend registered.
"""
from __future__ import annotations

import os
import sys

_INSTALLED = {}


def install(sobench_pkg=None):
    """Patch ``sobench`` (imported if not given) in place; idempotent.  Returns the module."""
    if sobench_pkg is None:
        import sobench as sobench_pkg  # noqa: PLC0415 -- the reference, on sys.path
    if _INSTALLED.get(id(sobench_pkg)):
        return sobench_pkg
    import sobench.backend as sb
    import sobench.bench as bench

    from .backend import CudaBackend

    ref_make_backend = sb.make_backend
    ref_run_cell = bench.run_cell

    def make_backend(kind, chunk_size=sb.DEFAULT_CHUNK, workers=None):
        if kind == "cuda":
            return CudaBackend(chunk_size, workers)
        return ref_make_backend(kind, chunk_size, workers)

    def run_cell(config, size, backend_kind, rep):
        if backend_kind != "cuda":
            return ref_run_cell(config, size, backend_kind, rep)
        return _run_cell_cuda(config, size, rep, bench)

    ref_run_bench = bench.run_bench

    def run_bench(config):
        written = ref_run_bench(config)
        if "cuda" in config.backends:  # the per-kernel roofline columns of the cuda cells
            path = os.path.join(config.out, "kernels.csv")
            write_kernel_csv(config, path)
            written.append(path)
        return written

    sb.make_backend = make_backend
    bench.make_backend = make_backend
    bench.run_cell = run_cell
    bench.run_bench = run_bench
    import sobench.cli as cli  # noqa: PLC0415 -- it imported run_bench by name
    cli.run_bench = run_bench
    if hasattr(sobench_pkg, "make_backend"):
        sobench_pkg.make_backend = make_backend
    _unify_errors()
    _route_functions()
    _INSTALLED[id(sobench_pkg)] = True
    return sobench_pkg


_ERROR_NAMES = ("SobenchError", "DimensionMismatch", "ConfigurationError", "EmptyRequest",
                "InsufficientSamples", "InvalidGradient", "InvalidConstraint", "SolverStall",
                "UndefinedMetric", "DegeneratePair", "RunAborted")


def _unify_errors():
    """Make what the device path raises catchable as sobench's exceptions (errors.py:4-53).

    For every class, a subclass of both ours and sobench's (same name) replaces ours in
    this package's modules and in the status-code table, so ``except
    sobench.errors.RunAborted`` in reference code and ``except
    paper_2404_11631_b200.errors.RunAborted`` both catch it.  (Python's ``except``
    matches the real class hierarchy; virtual subclasses do not count.)"""
    import sobench.errors as se

    from . import errors as oe
    if issubclass(oe.RunAborted, se.RunAborted):
        return
    new = {}
    for name in _ERROR_NAMES:
        ours, ref = getattr(oe, name), getattr(se, name)
        bases = (ours, ref) if name == "SobenchError" else (ours, new[oe.SobenchError], ref)
        new[ours] = type(name, bases, {"__module__": oe.__name__, "__doc__": ours.__doc__})
    dev = oe.DeviceError
    new[dev] = type("DeviceError", (dev, new[oe.SobenchError]),
                    {"__module__": oe.__name__, "__doc__": dev.__doc__})
    for mod in list(sys.modules.values()):
        if not getattr(mod, "__name__", "").startswith(__package__ or "paper_2404_11631_b200"):
            continue
        for attr, val in list(vars(mod).items()):
            if isinstance(val, type) and val in new:
                setattr(mod, attr, new[val])
            elif isinstance(val, dict) and any(isinstance(v, type) and v in new for v in val.values()):
                for k, v in list(val.items()):
                    if isinstance(v, type) and v in new:
                        val[k] = new[v]


# ---------------------------------------------------------------------------
# The reference's task, sampling and SQN functions take a backend argument; given the
# cuda backend they run this package's device implementation (the reference's numba
# kernels reach the CPU through backend.run_blocks, which the cuda backend refuses).
# Arguments and results are converted between the reference's dataclasses and ours.
def _our_stream(st):
    from .sampling import RngStream
    return RngStream(st.seed, st.stream_id, st.counter)


def _with_stream(fn, st, *args):
    """Run fn(our_stream, *args) and move the reference stream's counter along with it."""
    ours = _our_stream(st)
    out = fn(ours, *args)
    st.counter = ours.counter
    return out


def _our_spec(spec):
    from .sampling import GaussianSpec
    return GaussianSpec(mean=spec.mean, diag_std=spec.diag_std, chol_factor=spec.chol_factor)


def _our_data(data):
    from ._tensors import mat_dev, vec_dev
    from .sampling import ClassificationData
    key = (id(data), id(data.features), id(data.labels))
    hit = _DATA_CACHE.get(id(data))
    if hit is not None and hit[0] == key:
        return hit[1]
    ours = ClassificationData(features=mat_dev(data.features), labels=vec_dev(data.labels),
                              true_weights=data.true_weights)
    if len(_DATA_CACHE) >= 4:  # a few recent data sets (an SQN run reuses one many times)
        _DATA_CACHE.pop(next(iter(_DATA_CACHE)))
    _DATA_CACHE[id(data)] = (key, ours, data)  # keeps `data` alive while cached
    return ours


_DATA_CACHE = {}


def _our_sample_set(ss):
    from ._tensors import mat_dev, vec_dev
    from .tasks import MeanVarSampleSet
    return MeanVarSampleSet(mat_dev(ss.samples), vec_dev(ss.mean), ss.count)


def _ref_record(rec):
    import sobench.records as sr
    return sr.RunRecord(task=rec.task, size=rec.size, backend=rec.backend, rep=rec.rep, seed=rec.seed,
                        iterations=rec.iterations, objectives=rec.objectives,
                        elapsed_ns=rec.elapsed_ns, final_iterate=rec.final_iterate,
                        warnings=list(rec.warnings))


def _is_cuda(backend):
    return getattr(backend, "kind", None) == "cuda"


def _route_functions():
    import sobench.sampling as ss_
    import sobench.sqn as sq
    import sobench.tasks as st

    from . import sampling as os_
    from . import sqn as oq
    from . import tasks as ot
    from ._tensors import to_host

    def route(mod, name, backend_pos, impl):
        ref = getattr(mod, name)
        if getattr(ref, "_simopt_routed", False):
            return

        def fn(*args, **kwargs):
            backend = kwargs.get("backend", args[backend_pos] if len(args) > backend_pos else None)
            if _is_cuda(backend):
                return impl(*args, **kwargs)
            return ref(*args, **kwargs)
        fn.__name__, fn.__doc__, fn.__wrapped__ = ref.__name__, ref.__doc__, ref
        fn._simopt_routed = True
        # rebind the name in every sobench module that imported it
        import sys as _sys
        for m in list(_sys.modules.values()):
            if getattr(m, "__name__", "").startswith("sobench") and getattr(m, name, None) is ref:
                setattr(m, name, fn)

    route(ss_, "uniform01", 2, lambda stream, n, backend=None: _with_stream(os_.uniform01, stream, n))
    route(ss_, "standard_normal", 2,
          lambda stream, n, backend=None: _with_stream(os_.standard_normal, stream, n))
    route(ss_, "sample_returns", 3, lambda spec, n, stream, backend=None: _with_stream(
        lambda s_, sp, n_: os_.sample_returns(sp, n_, s_), stream, _our_spec(spec), n))
    route(ss_, "sample_demands", 4, lambda mu, sigma, n, stream, backend=None: _with_stream(
        lambda s_, m, sg, n_: ot.sample_demands(m, sg, n_, s_), stream, mu, sigma, n))

    def synth(n, stream, backend=None):
        data = _with_stream(lambda s_, n_: os_.synth_classification(n_, s_), stream, n)
        return ss_.ClassificationData(features=to_host(data.features), labels=to_host(data.labels),
                                      true_weights=to_host(data.true_weights))
    route(ss_, "synth_classification", 2, synth)

    def build(samples, backend):
        ours = ot.build_sample_set(samples, backend)
        return st.MeanVarSampleSet(samples=to_host(ours.samples), mean=to_host(ours.mean),
                                   centered=to_host(ours.centered), count=ours.count)
    route(st, "build_sample_set", 1, build)
    route(st, "mv_objective", 2, lambda w, ss, backend: ot.mv_objective(w, _our_sample_set(ss), backend))
    route(st, "mv_gradient", 2, lambda w, ss, backend: ot.mv_gradient(w, _our_sample_set(ss), backend))
    route(st, "nv_gradient_hat", 3, ot.nv_gradient_hat)
    route(st, "nv_gradient_exact", 2, ot.nv_gradient_exact)
    route(st, "nv_objective_exact", 2, ot.nv_objective_exact)
    route(st, "logistic_loss", 3, lambda w, data, idx, backend: ot.logistic_loss(w, _our_data(data), idx, backend))
    route(st, "logistic_gradient", 3,
          lambda w, data, idx, backend: ot.logistic_gradient(w, _our_data(data), idx, backend))
    route(st, "logistic_hvp", 4,
          lambda w, v, data, idx, backend: ot.logistic_hvp(w, v, _our_data(data), idx, backend))

    def hupd(pairs, t, memory, backend):
        ours = [oq.CorrectionPair(p.s, p.y, p.curvature) for p in pairs]
        return to_host(oq.hessian_update(ours, t, memory, backend))
    route(sq, "hessian_update", 3, hupd)

    def sqn(task, config, backend, *, task_label="classification", size=None, rep=0):
        cfg = oq.SqnConfig(config.pair_every, config.memory, config.beta, config.grad_batch,
                           config.hess_batch, config.iterations, _our_stream(config.stream))
        try:
            rec = oq.sqn_run(ot.LogisticTask(_our_data(task.data)), cfg, backend, task_label=task_label,
                             size=size, rep=rep)
        except Exception as exc:  # RunAborted: hand the reference's record type back
            partial = getattr(exc, "partial_record", None)
            if partial is not None:
                exc.partial_record = _ref_record(partial)
            raise
        finally:
            config.stream.counter = cfg.stream.counter
        return _ref_record(rec)
    route(sq, "sqn_run", 2, sqn)


def _run_cell_cuda(config, size, rep, bench):
    """bench.run_cell for the cuda backend: same cell, same streams, device path."""
    from .backend import CudaBackend
    from .frank_wolfe import FwConfig, fw_run
    from .instances import gen_meanvar_instance, gen_newsvendor_instance
    from .sampling import RngStream, synth_classification
    from .sqn import SqnConfig, sqn_run
    from .tasks import LogisticTask, MeanVarProblem, NewsvendorProblem

    backend = CudaBackend(config.chunk_size)
    instance_stream = RngStream(config.seed, bench.INSTANCE_STREAM)
    opt_stream = RngStream(config.seed, bench.FIRST_REP_STREAM + rep)
    if config.task == "classification":
        task = LogisticTask(synth_classification(size, instance_stream))
        cfg = SqnConfig(pair_every=config.sqn_pair_every, memory=config.sqn_memory,
                        beta=config.sqn_beta, grad_batch=config.sqn_grad_batch,
                        hess_batch=config.sqn_hess_batch, iterations=config.iterations,
                        stream=opt_stream)
        return sqn_run(task, cfg, backend, task_label="classification", size=size, rep=rep)
    if config.task == "meanvar":
        problem = MeanVarProblem(gen_meanvar_instance(size, instance_stream), backend)
    else:
        problem = NewsvendorProblem(gen_newsvendor_instance(size, instance_stream), backend)
    fw_cfg = FwConfig(epochs=config.iterations // config.resample_every,
                      inner_iters=config.resample_every,
                      sample_size=config.sample_size_for(size), stream=opt_stream,
                      sample_schedule=config.sample_schedule)
    return fw_run(problem, fw_cfg, backend, task_label=config.task, size=size, rep=rep)


KERNEL_HEADER = ["task", "size", "kernel", "launches", "mean_us", "algorithmic_bytes",
                 "achieved_GBps", "peak_GBps", "frac_of_hbm", "bound", "basis"]


def _hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs of this pool's B200s (repo root), else the copy-bandwidth
    fallback of the profiling recipe."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def _event_us(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    return best


def kernel_rows(config, size):
    """Roofline columns of the dominant kernels of one cuda cell (task, size): each kernel
    timed alone with CUDA events at the cell's shapes, algorithmic bytes in the reference's
    data model (fp64 scenarios, demands and features)."""
    from .backend import CudaBackend
    from .fused import MV, fused_rows
    from .instances import gen_meanvar_instance, gen_newsvendor_instance
    from .sampling import RngStream, synth_classification
    from .tasks import MeanVarProblem, NewsvendorProblem
    import torch
    peak = _hbm_peak()
    b = CudaBackend(config.chunk_size)
    rows = []

    def row(kernel, us, nbytes, bound, basis):
        gbs = nbytes / (us * 1e-6) / 1e9
        rows.append([config.task, size, kernel, 1, f"{us:.3f}", nbytes, f"{gbs:.1f}", f"{peak:.1f}",
                     f"{gbs / peak:.4f}", bound, basis])

    if config.task == "newsvendor":
        S = config.sample_size_for(size)
        prob = NewsvendorProblem(gen_newsvendor_instance(size, RngStream(config.seed, 0)), b)
        st = RngStream(config.seed, 2)
        row("k_nv_resample_ws", _event_us(lambda: prob.resample(st, S)), 8 * size * S,
            "issue (heavy-FMA pipe: Philox4x64-10)", "8 B per demand draw (the sorted fp64 matrix)")
    elif config.task == "meanvar":
        n = config.sample_size_for(size)
        prob = MeanVarProblem(gen_meanvar_instance(size, RngStream(config.seed, 0)), b, fused=True)
        st = RngStream(config.seed, 2)
        row("k_normal<affine> + exact mean", _event_us(lambda: prob.resample(st, n)), 8 * n * size,
            "fp64 issue (glibc-exact Box-Muller)", "8 B per return draw written")
        ss = prob.sample_set
        w = torch.full((size,), 1.0 / size, dtype=torch.float64, device="cuda")
        g = torch.empty(size, dtype=torch.float64, device="cuda")
        q = torch.empty(1, dtype=torch.float64, device="cuda")
        row("k_fused_rows<MV>", _event_us(lambda: fused_rows(MV, ss.samples, w, center=ss.mean,
                                                              col_scale=1.0 / (n - 1), col_out=g,
                                                              scalar_out=q)),
            8 * n * size, "hbm", "8 B per element of X (one read per FW iteration)")
    else:  # classification: the SQN's full-data loss pass (exact row dots)
        data = synth_classification(size, RngStream(config.seed, 0))
        x = torch.full((size,), 1.0 / size, dtype=torch.float64, device="cuda")
        feats = data.features
        n = feats.shape[0]
        row("k_matvec_rows (exact loss pass)", _event_us(lambda: b.matvec_device(feats, x)), 8 * n * size,
            "hbm / latency", "8 B per feature element")
    return rows


def write_kernel_csv(config, path):
    """kernels.csv beside the reference's summary.csv: one row per (task, size, kernel)."""
    import csv
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(KERNEL_HEADER)
        for size in config.sizes:
            for r in kernel_rows(config, size):
                w.writerow(r)


def main(argv=None) -> int:
    """The reference CLI (sobench.cli.main) with the cuda backend registered (the reference
    is taken from sys.path, else from the repo's baseline/_ref install)."""
    try:
        import sobench  # noqa: F401,PLC0415
    except ImportError:
        ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
        sys.path.insert(0, ref)
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_simopt")
    install()
    from sobench import cli
    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
