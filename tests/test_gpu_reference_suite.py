"""The REFERENCE's own test modules, run against the cuda backend.

baseline/_ref/tests is the reference's test directory (pkg/tests), copied next to its
install by __graft_entry__.build(); tests/sobench_cuda_plugin.py patches the reference
before collection (see its docstring).  Two runs:

* mode "cuda": the reference's "sequential" and "parallel" backends are both the cuda
  backend -- every test body (hand values, oracles, finite differences, error
  contracts, RunAborted identity) runs the device path; the LMO names run the device
  LMOs;
* mode "mixed": "parallel" is the cuda backend, "sequential" the reference CPU backend --
  the reference's own SEQ-vs-PAR bit-equality tests compare the device to the reference.

Tests that measure or assume the CPU thread pool itself are excluded (listed below).
"""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFTESTS = os.path.join(ROOT, "baseline", "_ref", "tests")
MODULES = ["test_backend.py", "test_tasks.py", "test_frank_wolfe.py", "test_lmo.py", "test_sqn.py",
           "test_sampling.py"]
# the CPU thread pool's speed-up (a ParallelBackend property, not an arithmetic contract)
EXCLUDED = ["test_backend.py::test_parallel_kernel_speedup"]


@pytest.mark.skipif(not os.path.isdir(REFTESTS), reason="reference tests not copied (run build())")
@pytest.mark.parametrize("mode", ["cuda", "mixed"])
def test_reference_suite_on_cuda(mode):
    args = [sys.executable, "-m", "pytest", *[os.path.join(REFTESTS, m) for m in MODULES],
            "-p", "tests.sobench_cuda_plugin", "-q", "-m", "not slow", "-p", "no:cacheprovider",
            *[x for e in EXCLUDED for x in ("--deselect", os.path.join(REFTESTS, e))]]
    env = dict(os.environ, SIMOPT_SOBENCH_MODE=mode, PYTHONPATH=ROOT)
    out = subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = out.stdout[-4000:]
    log = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(log):  # evidence for profiles/ when run on the GPU box
        with open(os.path.join(log, f"reference_suite_{mode}.txt"), "w") as fh:
            fh.write(out.stdout + out.stderr)
    assert out.returncode == 0, tail + out.stderr[-2000:]
    m = re.search(r"(\d+) passed", tail)
    assert m and int(m.group(1)) > 100, tail
    used = re.search(r"cuda_backends=(\d+) libsimopt_loaded=True", tail)
    assert used and int(used.group(1)) > 0, tail
