"""pytest plugin: run the REFERENCE's own test modules against the cuda backend.

    python -m pytest baseline/_ref/tests/test_backend.py ... -p tests.sobench_cuda_plugin

(tests/test_gpu_reference_suite.py does this; baseline/_ref/tests is the reference's
test directory, copied next to its install by __graft_entry__.build()).  At start-up,
before the modules are collected, the reference is patched with
paper_2404_11631_b200.sobench_plugin.install() -- "cuda" registered, the task,
sampling and SQN functions routed to the device path for the cuda backend, the
exception classes unified -- and its backend factory is rebound:

  SIMOPT_SOBENCH_MODE=cuda   both "sequential" and "parallel" build the cuda backend:
                             every test body runs the device path;
  SIMOPT_SOBENCH_MODE=mixed  "parallel" builds the cuda backend, "sequential" stays the
                             reference CPU backend: the reference's SEQ-vs-PAR
                             bit-equality tests compare the device against the reference.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
STATS = {"mode": None, "cuda_backends": 0}


def pytest_terminal_summary(terminalreporter):
    """Evidence that the device path ran: backends built and device kernels launched."""
    from paper_2404_11631_b200 import _lib
    lib = _lib._lib
    terminalreporter.write_line(
        f"sobench_cuda_plugin: mode={STATS['mode']} cuda_backends={STATS['cuda_backends']} "
        f"libsimopt_loaded={lib is not None}")


def pytest_configure(config):
    config.addinivalue_line("markers", "slow: long-running (reference marker)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_simopt")
    for p in (REF, ROOT):
        if p not in sys.path:
            sys.path.insert(0, p)
    import sobench
    import sobench.backend as sb

    from paper_2404_11631_b200.backend import CudaBackend
    from paper_2404_11631_b200.sobench_plugin import install
    install(sobench)
    mode = os.environ.get("SIMOPT_SOBENCH_MODE", "cuda")
    ref_make = sb.make_backend

    def cuda(chunk_size=sb.DEFAULT_CHUNK, workers=None):
        STATS["cuda_backends"] += 1
        return CudaBackend(chunk_size, workers)

    def make_backend(kind, chunk_size=sb.DEFAULT_CHUNK, workers=None):
        if kind == "parallel" or (mode == "cuda" and kind == "sequential"):
            return cuda(chunk_size, workers)
        return ref_make(kind, chunk_size, workers)

    sb.make_backend = make_backend
    sb.ParallelBackend = cuda
    if mode == "cuda":
        sb.SequentialBackend = lambda chunk_size=sb.DEFAULT_CHUNK: cuda(chunk_size)
    STATS["mode"] = mode
    if mode == "cuda":
        _route_lmos()


def _route_lmos():
    """The LMOs take no backend: in cuda mode the reference's own names call the device
    kernels (csrc/fw.cu, csrc/lp.cu) for every test that imports them."""
    import sobench.lmo as sl

    from paper_2404_11631_b200 import lmo as ol
    cache = {}

    def poly(p):
        key = id(p)
        if key not in cache or cache[key][0] is not p:
            cache[key] = (p, ol.PolytopeSet(p.A, p.C))
        return cache[key][1]

    routed = {
        "lmo_simplex_slack": ol.lmo_simplex_slack,
        "lmo_single_budget": ol.lmo_single_budget,
        "lmo_general": lambda g, polytope, max_iters=None: ol.lmo_general(g, poly(polytope), max_iters),
    }
    for m in list(sys.modules.values()):
        if getattr(m, "__name__", "").startswith("sobench"):
            for name, fn in routed.items():
                if getattr(m, name, None) is getattr(sl, name):
                    setattr(m, name, fn)
    for name, fn in routed.items():
        setattr(sl, name, fn)
