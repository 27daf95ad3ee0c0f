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
  ``summarize`` consume as they are.

    python -m paper_2404_11631_b200.sobench_plugin run --task newsvendor --sizes 1000 \\
        --backend cuda,parallel --reps 3

runs the reference CLI (sobench/cli.py) with the cuda backend registered.
"""
from __future__ import annotations

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

    sb.make_backend = make_backend
    bench.make_backend = make_backend
    bench.run_cell = run_cell
    if hasattr(sobench_pkg, "make_backend"):
        sobench_pkg.make_backend = make_backend
    _INSTALLED[id(sobench_pkg)] = True
    return sobench_pkg


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


def main(argv=None) -> int:
    """The reference CLI (sobench.cli.main) with the cuda backend registered."""
    install()
    from sobench import cli
    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
