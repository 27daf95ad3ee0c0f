"""The cuda backend registered inside the reference package (paper_2404_11631_b200.sobench_plugin).

The reference is the install in baseline/_ref (build() puts it there); its own run_cell /
run_bench / CSV writers drive the device path.  CPU tests check the registration and the
loud failure without a GPU; GPU tests compare whole cells against the reference's own
sequential backend on the same streams.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def sob():
    if not os.path.isdir(os.path.join(REF, "sobench")):
        pytest.skip("reference not installed in baseline/_ref (run __graft_entry__.build())")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_simopt")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import sobench
    from paper_2404_11631_b200.sobench_plugin import install
    return install(sobench)


def test_registration(sob):
    import sobench.backend as sb
    import sobench.bench as bench
    from sobench.errors import ConfigurationError
    assert sb.make_backend("sequential").kind == "sequential"
    with pytest.raises(ConfigurationError):
        sb.make_backend("gpu")                      # the reference's own test keeps holding
    import torch
    if not torch.cuda.is_available():
        from paper_2404_11631_b200.errors import DeviceError
        with pytest.raises(DeviceError):            # no silent CPU fallback
            bench.make_backend("cuda")


@pytest.mark.gpu
@pytest.mark.parametrize("task,size", [("meanvar", 120), ("newsvendor", 200), ("classification", 20)])
def test_cells_match_reference(sob, task, size):
    import sobench.bench as bench
    iters = 50 if task != "classification" else 40
    cfg = bench.BenchConfig(task=task, sizes=[size], backends=["cuda", "sequential"], reps=1,
                            iterations=iters, resample_every=25 if task != "classification" else 25,
                            sample_size=300 if task != "classification" else None)
    ours = bench.run_cell(cfg, size, "cuda", 0)
    ref = bench.run_cell(cfg, size, "sequential", 0)
    assert ours.backend == "cuda" and ref.backend == "sequential"
    assert np.array_equal(ours.iterations, ref.iterations)
    assert np.array_equal(np.asarray(ours.final_iterate), np.asarray(ref.final_iterate))
    assert np.array_equal(ours.objectives, ref.objectives)  # newsvendor too: glibc-exact erf


@pytest.mark.gpu
def test_run_bench_writes_reference_csv(sob, tmp_path):
    import sobench.bench as bench
    cfg = bench.BenchConfig(task="newsvendor", sizes=[100], backends=["cuda"], reps=2,
                            iterations=25, sample_size=200, out=str(tmp_path))
    bench.run_bench(cfg)
    names = os.listdir(tmp_path)
    assert "trace_newsvendor_100_cuda_rep0.csv" in names and "trace_newsvendor_100_cuda_rep1.csv" in names
    assert "kernels.csv" in names  # the per-kernel roofline columns of the cuda cells


@pytest.mark.gpu
@pytest.mark.parametrize("task,size", [("meanvar", 120), ("newsvendor", 100), ("classification", 20)])
def test_kernel_roofline_csv(sob, tmp_path, task, size):
    """kernels.csv: one row per dominant kernel of each cuda cell, with
    its CUDA-event time, algorithmic bytes and fraction of the measured HBM peak."""
    import csv
    import sobench.bench as bench
    from paper_2404_11631_b200.sobench_plugin import KERNEL_HEADER
    cfg = bench.BenchConfig(task=task, sizes=[size], backends=["cuda"], reps=1, iterations=25,
                            sample_size=200, out=str(tmp_path))
    bench.run_bench(cfg)
    with open(os.path.join(tmp_path, "kernels.csv")) as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == KERNEL_HEADER and len(rows) >= 2
    for r in rows[1:]:
        assert r[0] == task and int(r[1]) == size and float(r[4]) > 0 and int(r[5]) > 0
        assert 0 < float(r[8]) < 2


def test_errors_unified(sob):
    """After install(), what the device path raises is also sobench's exception class."""
    import sobench.errors as se
    import paper_2404_11631_b200.errors as oe
    from paper_2404_11631_b200 import _lib
    for name in ("DimensionMismatch", "ConfigurationError", "EmptyRequest", "InsufficientSamples",
                 "InvalidGradient", "InvalidConstraint", "SolverStall", "DegeneratePair", "RunAborted"):
        assert issubclass(getattr(oe, name), getattr(se, name)), name
    assert issubclass(oe.DeviceError, se.SobenchError)
    for code, cls in _lib.STATUS_TO_ERROR.items():
        assert issubclass(cls, se.SobenchError), code
    with pytest.raises(se.RunAborted) as ei:
        raise oe.RunAborted("x", partial_record="p")
    assert ei.value.partial_record == "p"


def test_run_blocks_refuses_host_callbacks(sob):
    """No silent CPU fallback: the cuda backend never runs the reference's numba callbacks."""
    import sobench.errors as se
    from paper_2404_11631_b200.backend import CudaBackend
    b = CudaBackend.__new__(CudaBackend)  # no device needed to check the refusal
    ran = []
    with pytest.raises(se.ConfigurationError):
        b.run_blocks(10, lambda lo, hi: ran.append((lo, hi)))
    assert ran == []
