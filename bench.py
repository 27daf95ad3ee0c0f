#!/usr/bin/env python
"""Benchmark: solver iterations/s per task at the largest d x n on B200 (BASELINE.json).

Headline line (the metric is quoted on BASELINE.json configs[1]):
  newsvendor C2, d = 10,000 products, S = 100,000 demand scenarios per epoch,
  M = 25 FW iterations per resampling epoch, fp64, seed 42 (instance stream
  (42,0), optimizer stream (42,2): sobench bench.py:40-41, :156-157).  One bench
  step = one resampling epoch = 1 resample (d*S Philox + Box-Muller draws) + 25 FW
  iterations; value = FW iterations/s.
`per_task` (same JSON line): every other task at its largest configured scale --
  C1 mean-variance FW d=10^3 N=10^4 (one GPU only), C3 logistic Newton-CG d=10^3
  N=10^6, C4 mean-variance FW d=2*10^4 N=10^6, C5 logistic explicit-Hessian Newton
  d=8192 N=10^7 -- each with its own value, roofline, clocks and (rank 0, N=1) CPU
  baseline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                  [--tasks c1,c3,c4,c5|none] [--dist-backend nccl|gloo]

--gpus N > 1 without a torchrun environment re-launches itself through
torch.distributed.run (one rank per GPU, 127.0.0.1 rendezvous).  C2 shards the
SAME problem's products (strong scaling): each rank draws and scans only its
products (Philox counter offset, no RNG communication); every FW step exchanges
the per-rank LMO argmins inside the step kernel over NVLink peer memory (CUDA IPC
mailboxes).  C3/C4/C5 shard the sample rows (strong scaling of the fixed N): the
d-vector sums cross ranks inside the fused pass's finish kernel over peer memory,
the C5 Hessian by one NCCL allreduce per Newton iteration.  DESIGN.md section 5.

--impl reference: the reference's own CPU implementation (sobench, installed in
baseline/_ref, numba ParallelBackend on every host core) at the SAME C2 config:
one fw_run of W + K full epochs, each epoch's time read from the run's own trace.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D, S, M, SEED = 10_000, 100_000, 25, 42
METRIC = "newsvendor Frank-Wolfe iterations/sec (d=10000, S=100000, M=25)"
TINY = {"D": 2_000, "S": 5_000}  # --tiny: the test-suite configuration (not a bench number)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tasks", default="c1,c3,c4,c5",
                    help="per_task entries besides the C2 headline (comma list, or none)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tiny", action="store_true",
                    help="test-suite sizes for every task (exercises the code paths only)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the N>1 path with several ranks on one GPU")
    return ap.parse_args()


def _free_port():
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def maybe_relaunch(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: re-exec as N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_setup(args):
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        ndev = max(torch.cuda.device_count(), 1)
        if args.dist_backend == "nccl" and ndev < world:
            raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, found {ndev}")
        dev = local % ndev
        torch.cuda.set_device(dev)
        if args.dist_backend == "nccl":
            # NCCL's init log (transport, NVLS) goes to a file per rank; rank 0 echoes
            # its communicator lines to stderr
            logdir = os.path.join("/tmp", f"simopt_nccl_{os.environ.get('MASTER_PORT', '0')}")
            os.makedirs(logdir, exist_ok=True)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
            os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(logdir, "nccl.%h.%p.log"))
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
        t = torch.ones(1, device="cuda" if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t)  # the communicator is up (NCCL creates it lazily otherwise)
        if rank == 0 and args.dist_backend == "nccl":
            _echo_nccl_log()
    return rank, world


def _echo_nccl_log():
    path = os.environ.get("NCCL_DEBUG_FILE", "").replace("%h", socket.gethostname()).replace(
        "%p", str(os.getpid()))
    try:
        with open(path) as fh:
            lines = [ln.rstrip() for ln in fh
                     if any(k in ln for k in ("NCCL version", "Init COMPLETE", "NVLS", "nvls",
                                              "P2P/CUMEM", "comm 0x", "Connected all"))]
    except OSError:
        lines = [f"(no NCCL log at {path})"]
    for ln in lines[:12]:
        print(f"[nccl rank0] {ln}", file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled every 10 ms during the timed region.

    NVML (pynvml) is initialised before the region so the first sample lands at its
    start; a sample is also taken on entry and on exit, so even a short region has
    readings.  Falls back to `nvidia-smi -lms` when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown,
    # sw_power_cap (the order of Q's reason columns)
    BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            try:
                import torch
                nidx = torch.cuda._get_nvml_device_index(index)
            except Exception:  # noqa: BLE001 -- older torch: the visible index
                nidx = index
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(nidx)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self.nvml = pynvml
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi below
            self.nvml = None

    def _sample_nvml(self):
        nv = self.nvml
        sm = float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
        fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        bits = int(fn(self.handle))
        self.rows.append([str(sm), str(self.max_sm)] +
                         ["Active" if bits & b else "Not Active" for b in self.BITS])

    def _poll(self):
        while not self.stop.wait(0.01):
            try:
                self._sample_nvml()
            except Exception:  # noqa: BLE001
                return

    def __enter__(self):
        if self.nvml is not None:
            self._sample_nvml()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=1)
            try:
                self._sample_nvml()
            except Exception:  # noqa: BLE001
                pass
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def tensor_peaks():
    """Measured FP64-DMMA and tcgen05 kind::i8 peaks of this pool's B200s (not in
    MEASURED_PEAKS.json, which holds HBM and bf16 only): profiles/peaks_tensor.json."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_tensor.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {"fp64_dmma_tflops": 37.0, "i8_tcgen05_tops": 4500.0, "source": "fallback"}


def profiled_traffic():
    """DRAM bytes per k_nv_resample launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_inputs.json")) as fh:
            return json.load(fh).get("k_nv_resample", {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def _release():
    import torch
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU reference
def reference_available():
    return os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "sobench"))


def _sobench():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_simopt")
    p = os.path.join(ROOT, "baseline", "_ref")
    if p not in sys.path:
        sys.path.insert(0, p)
    import sobench
    from sobench import _kernels
    _kernels.warmup()  # JIT compilation stays out of every timed region (bench.py:154)
    return sobench


def reference_c2_epochs(n_epochs, d=D, s_=S, threads=None):
    """The reference's own C2 run: one sobench fw_run of n_epochs full epochs
    (frank_wolfe.py:91-121; each epoch = sample_demands incl. the row sort,
    sampling.py:173-193, + M FW iterations) on ParallelBackend with every host core.
    Returns each epoch's wall time, from the run's own trace stamps (a step's stamp
    is taken after its objective; epoch k spans the stamps of its last step and of
    the previous epoch's last step, so the resample is inside it)."""
    _sobench()
    from sobench.backend import make_backend
    from sobench.bench import gen_newsvendor_instance
    from sobench.frank_wolfe import FwConfig, fw_run
    from sobench.sampling import RngStream
    from sobench.tasks import NewsvendorProblem
    threads = threads or os.cpu_count() or 1
    b = make_backend("parallel", workers=threads)
    task = gen_newsvendor_instance(d, RngStream(SEED, 0))
    rec = fw_run(NewsvendorProblem(task, b), FwConfig(n_epochs, M, s_, RngStream(SEED, 2)), b)
    ends = [0] + [int(rec.elapsed_ns[(k + 1) * M - 1]) for k in range(n_epochs)]
    return [(ends[k + 1] - ends[k]) / 1e9 for k in range(n_epochs)], threads, rec


def port_c2_epochs(n_epochs, d=D, s_=S):
    """No reference installed: the C oracle port (single thread), same run."""
    from oracle import oracle as orc
    task = orc.gen_newsvendor_instance(d, orc.Stream(SEED, 0))
    out = []
    st = orc.Stream(SEED, 2)
    for _ in range(n_epochs):  # epochs of one run continue the stream; x restarts (same work)
        t = time.perf_counter()
        orc.fw_run_newsvendor(task, 1, M, s_, st)
        out.append(time.perf_counter() - t)
    return out, 1


def cpu_baseline_c2(dd, ss):
    if reference_available():
        ts, cores, _ = reference_c2_epochs(1, dd, ss)
        kind = "reference"
    else:
        ts, cores = port_c2_epochs(1, dd, ss)
        kind = "port"
    t = ts[0]
    return {"value": M / t, "unit": "iterations/s", "cores": cores, "kind": kind,
            "sample": (f"1 full C2 epoch (d={dd}, resample S={ss} incl. row sort + {M} FW "
                       f"iterations) through sobench fw_run, ParallelBackend, {t:.2f} s"
                       if kind == "reference" else
                       f"1 full C2 epoch (d={dd}, S={ss}) via the C oracle port, {t:.2f} s")}


def run_reference(args, rank):
    if rank != 0:
        return
    dd, ss = (TINY["D"], TINY["S"]) if args.tiny else (D, S)
    n = args.warmup + args.steps
    if reference_available():
        ts, cores, rec = reference_c2_epochs(n, dd, ss)
        kind = "reference"
        final = float(rec.objectives[-1])
    else:
        ts, cores = port_c2_epochs(n, dd, ss)
        kind, final = "port", None
    timed = ts[args.warmup:]
    per_step = statistics.mean(timed)
    value = M / per_step
    line = {
        "impl": "reference", "metric": _metric(args, dd, ss),
        "value": value, "unit": "iterations/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _c2_config(args, dd, ss, 1),
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores, "kind": kind,
                         "sample": (f"one sobench fw_run of {n} full epochs (d={dd}, S={ss}, M={M}); "
                                    f"the last {args.steps} epochs timed from the run's trace "
                                    "stamps" if kind == "reference" else
                                    f"{n} full epochs of the C oracle port, last {args.steps} timed")},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "final_objective": final,
    }
    print(json.dumps(line), flush=True)


def _metric(args, dd, ss):
    return METRIC if not args.tiny else f"TINY newsvendor FW iterations/sec (d={dd}, S={ss}, M={M})"


def _c2_config(args, dd, ss, world):
    return {"workload": ("newsvendor C2 (BASELINE.json configs[1])" if not args.tiny else
                         "TINY test configuration (not the C2 bench)"),
            "d": dd, "S": ss, "M": M, "seed": SEED,
            "step": f"1 resampling epoch = 1 resample + {M} FW iterations",
            "timing": ("steady-state pipeline: the timed region holds K resample launches and K "
                       "epochs of FW steps, each epoch's steps overlapping the next epoch's resample"),
            "l2": "inputs larger than L2 (8 GB of fp64 demands per epoch in the reference's data "
                  "model; 4.5 GB of keyed layout here)",
            "parallelism": (f"products sharded x{world}" if world > 1 else "single GPU")}


# ---------------------------------------------------------------- ours: C2 headline
def philox_floor(nblocks, kernel_ms):
    """The resample's arithmetic floor, timed in this run: the same Philox4x64-10 core over
    the launch's blocks with nothing stored (simopt_philox_floor), CUDA events."""
    import torch
    from paper_2404_11631_b200 import _lib
    out = torch.empty(8 * torch.cuda.get_device_properties(0).multi_processor_count * 256,
                      dtype=torch.int64, device="cuda")
    call = lambda: _lib.call("simopt_philox_floor", _lib.stream_ptr(), SEED, 2, 0, nblocks,
                             _lib.ptr(out), out.numel())
    call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(3):
        e0.record()
        call()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    floor = min(times)
    return {"bound": "issue: heavy-FMA pipe (IMAD.WIDE of the Philox 64x64->128 products)",
            "floor_ms": floor, "kernel_ms": kernel_ms, "frac": floor / kernel_ms,
            "basis": f"Philox4x64-10 of the launch's {nblocks} blocks through the resample's own "
                     "17-product core with nothing stored, timed in this run"}


def run_c2(args, rank, world, shard):
    import torch
    import paper_2404_11631_b200 as pkg
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.records import TraceBuilder
    from paper_2404_11631_b200.tasks import NewsvendorProblem, make_nv_engine, nv_geometry

    dd, ss = (TINY["D"], TINY["S"]) if args.tiny else (D, S)
    backend = pkg.make_backend("cuda")
    task = gen_newsvendor_instance(dd, pkg.RngStream(SEED, 0))
    prob = NewsvendorProblem(task, backend, shard=shard)
    epochs = args.warmup + args.steps
    eng = make_nv_engine(prob, M, epochs, backend.chunk_size)  # CUDA-graph epochs when sharded
    stream = pkg.RngStream(SEED, 2)
    eng.start()
    # steady-state pipeline: every epoch's steps overlap the next epoch's resample.  The
    # timed region holds exactly K resample launches and K epochs of steps: the first timed
    # epoch's resample is the warm-up's last overlap, the resample behind the last timed
    # epoch runs inside the region.
    for k in range(args.warmup):
        eng.enqueue_epoch(k, stream, ss, next_samples=ss)
    eng.finish()
    torch.cuda.synchronize()
    if shard is not None:
        shard.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record()
        for k in range(args.warmup, epochs):
            eng.enqueue_epoch(k, stream, ss, time_resample=True, next_samples=ss)
        eng.finish()
        e1.record()
        torch.cuda.synchronize()
    if shard is not None:
        shard.barrier()
    ms = _max_over_ranks(e0.elapsed_time(e1), world)
    # validate the whole run (trace rows, feasibility) outside the timed region
    trace = TraceBuilder()
    for k in range(epochs):
        bad = eng.check_epoch(k, trace)
        if bad:
            raise RuntimeError(f"bench run aborted at step {bad[0]}: {bad[1]}")
    value = args.steps * M / (ms / 1e3)  # one problem, all ranks (strong scaling)
    res_ms = statistics.mean(a.elapsed_time(b) for a, b in eng.resample_events)
    seg, nbuck = nv_geometry()
    nseg = -(-ss // seg)
    d_loc = prob.dev.d
    # the algorithmic bytes of a resample launch are the epoch's fp64
    # demand matrix written once, 8 B per draw (the reference's data model).  This
    # kernel actually writes 4 B keys + 2-byte bucket starts per 4096-draw segment
    # (keyed layout), measured as `traffic`.
    alg_bytes = d_loc * ss * 8
    stored_bytes = d_loc * ss * 4 + d_loc * nseg * nbuck * 2
    peak, peak_kind = peaks()
    achieved = alg_bytes / (res_ms / 1e3) / 1e9
    traffic = profiled_traffic()  # captured at N=1 (all d products): this rank's share
    if traffic is not None:
        traffic = int(round(traffic * d_loc / D))
    compute_roof = philox_floor(d_loc * ss // 4, res_ms)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "k_nv_resample", "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "algorithmic_bytes_per_launch": alg_bytes, "stored_bytes_per_launch": stored_bytes,
                "kernel_ms": res_ms, "share_of_step": res_ms / (ms / args.steps),
                "note": ("instruction-bound by design: Philox4x64-10 + an fp32 SFU Box-Muller key "
                         "per draw, exact glibc Box-Muller only for the few ambiguous draws at "
                         "query time; kernel_ms is measured (CUDA events on the generator stream) "
                         "while the previous epoch's FW steps run; see profiles/"),
                "compute_roof": compute_roof}
    # the step against SURVEY 8(d)'s per-iteration roof (8 d S (1 + 1/M) bytes: one scan of
    # the epoch's demands per gradient + the amortised write) -- the keyed ECDF reads a
    # window of buckets per product instead of all S demands, so it runs above that roof
    it_roof = peak * 1e9 * world / (8 * dd * ss * (1 + 1 / M))
    step_roofline = {"unit": "iterations/s", "data_model_roof": it_roof, "achieved": value,
                     "frac": value / it_roof,
                     "basis": "SURVEY 8(d) C2: 8*d*S*(1+1/M) bytes per FW iteration at hbm peak "
                              "(x n_gpus)"}
    launches_per_epoch = M + 4  # resample, M+1 fused steps (stamping themselves), records (terms + sums)
    if world > 1 and eng.mailbox is None:
        launches_per_epoch += 2 * M  # LMO pack + apply around each NCCL exchange
    cfg = _c2_config(args, dd, ss, world)
    if world > 1:
        cfg["parallelism"] += ("; per-step LMO exchange " +
                               ("inside the step kernel over NVLink peer memory (CUDA IPC)"
                                if eng.mailbox is not None else f"by {args.dist_backend} allgather"))
    line = {
        "metric": _metric(args, dd, ss),
        "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "roofline": roofline,
        "step_roofline": step_roofline,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_epoch * args.steps,
        "final_objective": trace.build("newsvendor", dd, "cuda", 0, SEED, None).final_objective,
    }
    del eng, prob
    _release()  # the headline run's layouts go back before the end-to-end run allocates its own
    if not args.no_e2e:
        line["e2e"] = run_e2e(task, backend, shard, ss)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_c2(dd, ss)
    return line


def run_e2e(task, backend, shard, ss):
    """Same metric through the public API with host inputs, the way the reference's
    run_cell (bench.py:152-184) runs a cell: build the problem from the host instance
    arrays (H2D of mu, sigma, k, h, v, c) and call fw_run for the reference's 60 epochs
    (1500 FW iterations, bench.py:88; one step = one resampling epoch).  Every epoch's draw
    state goes to the device with its launches and every epoch's trace rows (flags,
    feasibility sums, objectives, stamps) come back to the host for the reference's
    checks before the run continues; the RunRecord (trace + final iterate) is returned.
    Timed on the wall clock around the whole call, max over ranks."""
    import torch
    import paper_2404_11631_b200 as pkg
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.tasks import NewsvendorProblem
    steps = 60  # the reference bench's run length: 1500 FW iterations = 60 epochs (bench.py:88)
    dd = task.dimension
    fw_run(NewsvendorProblem(task, backend, shard=shard), FwConfig(2, M, ss, pkg.RngStream(SEED, 2)),
           backend)  # warm: allocations, layouts, streams
    gc.collect()  # a collection inside the timed call would stall the host's enqueue
    torch.cuda.synchronize()
    if shard is not None:
        shard.barrier()
    t = time.perf_counter()
    rec = fw_run(NewsvendorProblem(task, backend, shard=shard),
                 FwConfig(steps, M, ss, pkg.RngStream(SEED, 2)), backend)
    torch.cuda.synchronize()
    dt = _max_over_ranks(time.perf_counter() - t, 1 if shard is None else shard.world)
    assert rec.iterations.size == steps * M
    h2d = 6 * dd * 8 / steps + 4 * 8  # instance once per run (amortised) + the epoch's draw words
    d2h = M * (4 + 8 + 8 + 8) + dd * 8 / steps  # per-epoch trace rows + the final iterate (amortised)
    return {"value": steps * M / dt, "unit": "iterations/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "epochs": steps,
            "note": "one fw_run call of `epochs` epochs from host instance arrays (run_cell's call)"}


# ---------------------------------------------------------------- ours: per-task entries
def _timed_fw(prob, backend, n_samples, warm, timed, world, shard, stream):
    """fw_run of `warm` epochs, then of `timed` epochs between CUDA events (the same
    problem and a continuing stream), max over ranks.  Returns (ms, record, clocks)."""
    import torch
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    fw_run(prob, FwConfig(warm, M, n_samples, stream), backend)
    torch.cuda.synchronize()
    if shard is not None:
        shard.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record()
        rec = fw_run(prob, FwConfig(timed, M, n_samples, stream), backend)
        e1.record()
        torch.cuda.synchronize()
    return _max_over_ranks(e0.elapsed_time(e1), world), rec, clk.summary()


def _timed_newton(fn, warm, timed, world, shard):
    """One Newton run of warm + timed iterations; CUDA events recorded after each
    iteration's enqueue; the timed span is events[warm-1] -> events[warm+timed-1]."""
    import torch
    evs = []

    def hook(it):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        evs.append(e)
    if shard is not None:
        shard.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        rec = fn(warm + timed, hook)
        torch.cuda.synchronize()
    ms = evs[warm - 1].elapsed_time(evs[warm + timed - 1])
    return _max_over_ranks(ms, world), rec, clk.summary()


def task_c1(args, world, shard):
    import paper_2404_11631_b200 as pkg
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    d, N = (200, 2_000) if args.tiny else (1_000, 10_000)
    b = pkg.make_backend("cuda")
    prob = MeanVarProblem(gen_meanvar_instance(d, pkg.RngStream(SEED, 0)), b, fused=True)
    W, K = 3, 20
    ms, rec, clk = _timed_fw(prob, b, N, W, K, world, shard, pkg.RngStream(SEED, 2))
    it_s = K * M / (ms / 1e3)
    alg = 8 * N * d * (1 + 1 / M)
    peak, pk = peaks()
    return {"workload": "C1 mean-variance Frank-Wolfe (BASELINE.json configs[0])", "d": d, "N": N,
            "M": M, "mode": "fused single pass (trajectory within 1e-8 of the reference)",
            "metric": "FW iterations/s", "value": it_s, "unit": "iterations/s",
            "warmup_epochs": W, "epochs": K, "ms_per_epoch": ms / K, "n_gpus": 1,
            "l2": "one epoch's X (80 MB) is re-read by its 25 iterations and stays L2-resident, as "
                  "the algorithm dictates; each epoch draws a new X (two buffers, 160 MB > L2)",
            "roofline": {"bound": "hbm", "achieved": alg * it_s / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg * it_s / 1e9 / peak, "traffic": None,
                         "basis": "SURVEY 8(d) C1: 8 N d (1 + 1/M) algorithmic bytes per FW iteration",
                         "peak_kind": pk,
                         "note": ("one cooperative launch per epoch (simopt_mv_fw_epoch): latency-bound "
                                  "-- per step a pass over 80 MB of L2-resident X, two grid barriers, "
                                  "the column fold and the LMO tail")},
            "clocks": clk, "final_objective": float(rec.objectives[-1])}


def task_c3(args, world, shard):
    import paper_2404_11631_b200 as pkg
    from paper_2404_11631_b200.newton import newton_cg
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.tasks import LogisticTask
    d, N, kcg = (300, 20_000, 10) if args.tiny else (1_000, 1_000_000, 10)
    b = pkg.make_backend("cuda")
    W, K = 3, 20
    peak, pk = peaks()
    out = {"workload": "C3 logistic Newton-CG (BASELINE.json configs[2])", "d": d, "N": N,
           "k_cg": kcg, "metric": "Newton iterations/s", "unit": "iterations/s", "n_gpus": world,
           "scaling": "strong (rows sharded)" if world > 1 else None, "variants": []}
    for packed in (True, False):
        data = synth_classification(d, pkg.RngStream(SEED, 0), n_rows=N, shard=shard, packed=packed)
        task = LogisticTask(data)
        ms, rec, clk = _timed_newton(
            lambda n, hook: newton_cg(task, n, kcg, b, fused=True, on_iteration=hook), W, K, world, shard)
        it_s = K / (ms / 1e3)
        nl = data.local_rows
        alg = 8 * nl * d * (kcg + 1)          # fp64 X read k+1 times per iteration
        words = -(-d // 64)
        stored = 8 * nl * words * (kcg + 1) * (2 if d > 1024 else 1)
        v = {"features": "bit-packed (exact: X is 0/1)" if packed else "fp64", "value": it_s,
             "ms_per_iteration": ms / K, "warmup_iterations": W, "iterations": K,
             "clocks": clk, "final_objective": float(rec.objectives[-1]),
             "l2": "inputs larger than L2" if not packed or nl * words * 8 > 126e6 else
                   "bit-packed X fits L2"}
        if packed:
            v["roofline"] = {"bound": "issue", "achieved": stored * it_s / 1e9, "peak": peak,
                             "unit": "GB/s", "frac": stored * it_s / 1e9 / peak, "traffic": None,
                             "basis": "bytes of the bit-packed X read per iteration (k+1 passes)",
                             "data_model_GBps": alg * it_s / 1e9,
                             "data_model_frac": alg * it_s / 1e9 / peak,
                             "note": "nibble-table passes are ALU-issue-bound at 1/64 of the fp64 "
                                     "bytes; data_model_* is SURVEY 8(d)'s fp64 model (beats it)"}
        else:
            v["roofline"] = {"bound": "hbm", "achieved": alg * it_s / 1e9, "peak": peak,
                             "unit": "GB/s", "frac": alg * it_s / 1e9 / peak, "traffic": None,
                             "basis": "SURVEY 8(d) C3: 8 N d (k_CG + 1) bytes per Newton iteration",
                             "peak_kind": pk}
        out["variants"].append(v)
        del data, task
        _release()
    out["value"] = out["variants"][0]["value"]
    out["roofline"] = out["variants"][1]["roofline"]  # the HBM-bound fp64 pass, per GPU
    return out


def task_c4(args, world, shard):
    import paper_2404_11631_b200 as pkg
    from paper_2404_11631_b200.instances import gen_meanvar_instance
    from paper_2404_11631_b200.tasks import MeanVarProblem
    d, N = (400, 50_000) if args.tiny else (20_000, 1_000_000)
    b = pkg.make_backend("cuda")
    prob = MeanVarProblem(gen_meanvar_instance(d, pkg.RngStream(SEED, 0)), b, fused=True, shard=shard)
    W, K = 2, 3
    ms, rec, clk = _timed_fw(prob, b, N, W, K, world, shard, pkg.RngStream(SEED, 2))
    it_s = K * M / (ms / 1e3)
    nl = prob.sample_set.samples.shape[0]
    alg = 8 * nl * d * (1 + 1 / M)               # this GPU's algorithmic bytes per FW iteration
    peak, pk = peaks()
    out = {"workload": "C4 mean-variance Frank-Wolfe at scale (BASELINE.json configs[3])", "d": d,
           "N": N, "M": M, "rows_per_gpu": nl,
           "mode": "fused single pass (trajectory within 1e-8); cross-rank d+1 sums inside the "
                   "pass's finish kernel over NVLink peer memory" if world > 1 else
                   "fused single pass (trajectory within 1e-8)",
           "metric": "FW iterations/s", "value": it_s, "unit": "iterations/s", "n_gpus": world,
           "scaling": "strong (rows sharded)" if world > 1 else None,
           "warmup_epochs": W, "epochs": K, "ms_per_epoch": ms / K,
           "l2": "inputs larger than L2 (X is %.0f GB per GPU)" % (8 * nl * d / 1e9),
           "roofline": {"bound": "hbm", "achieved": alg * it_s / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": alg * it_s / 1e9 / peak, "traffic": None, "peak_kind": pk,
                        "basis": "SURVEY 8(d) C4: 8 N_gpu d (1 + 1/M) bytes per FW iteration per GPU "
                                 "(one fused read of X per step + the amortised draw)"},
           "clocks": clk, "final_objective": float(rec.objectives[-1])}
    try:  # the fused pass's cluster geometry on this chip (explains box-to-box spread)
        import torch
        from paper_2404_11631_b200.fused import MV, fused_geometry
        out["pass_geometry"] = dict(fused_geometry(MV, d), sms=torch.cuda.get_device_properties(0).multi_processor_count)
    except Exception as e:  # diagnostic only
        out["pass_geometry"] = {"error": str(e)}
    del prob
    _release()
    return out


def task_c5(args, world, shard):
    import paper_2404_11631_b200 as pkg
    from paper_2404_11631_b200.newton import newton_explicit
    from paper_2404_11631_b200.sampling import synth_classification
    from paper_2404_11631_b200.tasks import LogisticTask
    d, N, kcg = (1_100, 40_000, 20) if args.tiny else (8_192, 10_000_000, 20)
    b = pkg.make_backend("cuda")
    data = synth_classification(d, pkg.RngStream(SEED, 0), n_rows=N, shard=shard, packed=True)
    task = LogisticTask(data)
    W, K = 1, 3
    ms, rec, clk = _timed_newton(
        lambda n, hook: newton_explicit(task, n, kcg, b, on_iteration=hook), W, K, world, shard)
    it_s = K / (ms / 1e3)
    nl = data.local_rows
    tp = tensor_peaks()
    i8_ops = 5 * nl * d * (d + 1)          # five exact u8 limb GEMMs, SYRK convention
    fp64_eq = nl * d * (d + 1)             # SURVEY 8(d) C5 flops (SYRK convention)
    out = {"workload": "C5 logistic explicit-Hessian Newton (BASELINE.json configs[4])", "d": d,
           "N": N, "k_cg": kcg, "rows_per_gpu": nl,
           "mode": "bit-packed X (exact: X is 0/1); H = X^T D X as five exact 8-bit limb GEMMs "
                   "on tcgen05 (kind::i8, TMEM accumulators, TMA operands); CG on H"
                   + ("; one NCCL allreduce of the d x d Hessian per iteration" if world > 1 else ""),
           "metric": "Newton iterations/s", "value": it_s, "unit": "iterations/s", "n_gpus": world,
           "scaling": "strong (rows sharded)" if world > 1 else None,
           "warmup_iterations": W, "iterations": K, "ms_per_iteration": ms / K,
           "l2": "inputs larger than L2",
           "roofline": {"bound": "tensor", "achieved": i8_ops * it_s / 1e12,
                        "peak": tp["i8_tcgen05_tops"], "unit": "TOPS",
                        "frac": i8_ops * it_s / 1e12 / tp["i8_tcgen05_tops"], "traffic": None,
                        "basis": "5 N_gpu d (d+1) int8 tensor ops per Newton iteration (the whole "
                                 "iteration's time, Hessian ~95% of it)",
                        "peak_kind": f"measured tcgen05 kind::i8 rate ({tp.get('source')})",
                        "fp64_equivalent_tflops": fp64_eq * it_s / 1e12,
                        "fp64_dmma_peak_tflops": tp["fp64_dmma_tflops"],
                        "fp64_equivalent_frac_of_dmma_peak": fp64_eq * it_s / 1e12 / tp["fp64_dmma_tflops"]},
           "clocks": clk, "final_objective": float(rec.objectives[-1])}
    del data, task
    _release()
    return out


# ---------------------------------------------------------------- per-task CPU baselines
def cpu_c1(tiny):
    """The reference at full C1 size: one sobench fw_run epoch (resample + M iterations)."""
    if not reference_available():
        return None
    _sobench()
    from sobench.backend import make_backend
    from sobench.bench import gen_meanvar_instance
    from sobench.frank_wolfe import FwConfig, fw_run
    from sobench.sampling import RngStream
    from sobench.tasks import MeanVarProblem
    d, N = (200, 2_000) if tiny else (1_000, 10_000)
    threads = os.cpu_count() or 1
    b = make_backend("parallel", workers=threads)
    prob = MeanVarProblem(gen_meanvar_instance(d, RngStream(SEED, 0)), b)
    t = time.perf_counter()
    fw_run(prob, FwConfig(2, M, N, RngStream(SEED, 2)), b)
    t = (time.perf_counter() - t) / 2
    return {"value": M / t, "unit": "iterations/s", "cores": threads, "kind": "reference",
            "sample": f"2 full C1 epochs through sobench fw_run (ParallelBackend), {t:.2f} s/epoch"}


def cpu_c3(tiny):
    """One Newton-CG iteration at full C3 size from the reference's own building blocks
    (tasks.py:216-253: logistic_gradient + k_CG x logistic_hvp + logistic_loss; the
    oracle newton_cg's call sequence), ParallelBackend on every core."""
    if not reference_available():
        return None
    import numpy as np
    _sobench()
    from sobench.backend import make_backend
    from sobench.sampling import ClassificationData
    from sobench.tasks import logistic_gradient, logistic_hvp, logistic_loss
    d, N, kcg = (300, 20_000, 10) if tiny else (1_000, 1_000_000, 10)
    threads = os.cpu_count() or 1
    b = make_backend("parallel", workers=threads)
    rng = np.random.Generator(np.random.Philox(SEED))
    x = rng.integers(0, 2, size=(N, d), dtype=np.uint8).astype(np.float64)
    z = rng.integers(0, 2, size=N).astype(np.float64)
    data = ClassificationData(features=x, labels=z, true_weights=np.zeros(d))
    w = rng.standard_normal(d) * 0.01
    v = rng.standard_normal(d)
    t = time.perf_counter()
    logistic_gradient(w, data, None, b)
    for _ in range(kcg):
        logistic_hvp(w, v, data, None, b)
    logistic_loss(w, data, None, b)
    t = time.perf_counter() - t
    return {"value": 1 / t, "unit": "iterations/s", "cores": threads, "kind": "reference",
            "sample": f"1 full-size Newton-CG iteration (N={N}, d={d}): sobench logistic_gradient + "
                      f"{kcg} x logistic_hvp + logistic_loss, ParallelBackend, {t:.2f} s"}


def cpu_c4(tiny):
    """The reference's FW epoch at C4's d and a reduced N, scaled linearly in N
    (C4's fp64 X is 160 GB)."""
    if not reference_available():
        return None
    _sobench()
    from sobench.backend import make_backend
    from sobench.bench import gen_meanvar_instance
    from sobench.frank_wolfe import FwConfig, fw_run
    from sobench.sampling import RngStream
    from sobench.tasks import MeanVarProblem
    d, N, n_s = (400, 50_000, 5_000) if tiny else (20_000, 1_000_000, 5_000)
    threads = os.cpu_count() or 1
    b = make_backend("parallel", workers=threads)
    prob = MeanVarProblem(gen_meanvar_instance(d, RngStream(SEED, 0)), b)
    t = time.perf_counter()
    fw_run(prob, FwConfig(1, M, n_s, RngStream(SEED, 2)), b)
    t = time.perf_counter() - t
    scaled = t * N / n_s
    return {"value": M / scaled, "unit": "iterations/s", "cores": threads, "kind": "reference",
            "sample": f"1 sobench FW epoch at d={d}, N={n_s} ({t:.2f} s), scaled linearly to N={N}"}


def cpu_c5(tiny):
    """C5 has no reference function: the reference test's explicit Hessian
    ((x.T*(c*(1-c)))@x/N, tests/test_tasks.py:297-299) in numpy BLAS + sobench
    logistic_gradient at a reduced N, scaled linearly in N, + the CG solve (20 d x d
    matvecs, N-independent)."""
    import numpy as np
    d, N, n_s, kcg = (1_100, 40_000, 4_000, 20) if tiny else (8_192, 10_000_000, 20_000, 20)
    rng = np.random.Generator(np.random.Philox(SEED))
    x = rng.integers(0, 2, size=(n_s, d), dtype=np.uint8).astype(np.float64)
    z = rng.integers(0, 2, size=n_s).astype(np.float64)
    w = rng.standard_normal(d) * 0.01
    threads = os.cpu_count() or 1
    grad = None
    if reference_available():
        _sobench()
        from sobench.backend import make_backend
        from sobench.sampling import ClassificationData
        from sobench.tasks import logistic_gradient
        b = make_backend("parallel", workers=threads)
        data = ClassificationData(features=x, labels=z, true_weights=np.zeros(d))
        grad = lambda: logistic_gradient(w, data, None, b)  # noqa: E731
    t = time.perf_counter()
    c = 1.0 / (1.0 + np.exp(-(x @ w)))
    h = (x.T * (c * (1 - c))) @ x / n_s
    if grad is not None:
        grad()
    t_n = time.perf_counter() - t
    v = rng.standard_normal(d)
    t = time.perf_counter()
    for _ in range(kcg):
        v = h @ v
        v /= np.linalg.norm(v)
    t_cg = time.perf_counter() - t
    total = t_n * N / n_s + t_cg
    return {"value": 1 / total, "unit": "iterations/s", "cores": threads, "kind": "port",
            "sample": f"numpy BLAS explicit Hessian (the reference test's expression) + sobench "
                      f"logistic_gradient at N={n_s} ({t_n:.2f} s) scaled linearly to N={N}, + "
                      f"{kcg} CG matvecs ({t_cg:.2f} s)"}


CPU_TASKS = {"c1": cpu_c1, "c3": cpu_c3, "c4": cpu_c4, "c5": cpu_c5}
GPU_TASKS = {"c1": task_c1, "c3": task_c3, "c4": task_c4, "c5": task_c5}


def run_ours(args, rank, world):
    shard = None
    if world > 1:
        from paper_2404_11631_b200.sharding import ShardGroup
        shard = ShardGroup()
    line = run_c2(args, rank, world, shard)
    tasks = [t for t in args.tasks.split(",") if t and t != "none"]
    per = {}
    for name in tasks:
        if name == "c1" and world > 1:
            continue  # 10^4 scenarios: a one-GPU config (BASELINE.json configs[0])
        per[name] = GPU_TASKS[name](args, world, shard)
        _release()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        for name, ent in per.items():
            cb = CPU_TASKS[name](args.tiny)
            if cb is not None:
                ent["cpu_baseline"] = cb
    if per:
        line["per_task"] = per
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        # host-CPU arm: rank 0 alone times the reference; other ranks exit at once
        run_reference(args, int(os.environ.get("RANK", "0")))
        return
    maybe_relaunch(args)
    rank, world = dist_setup(args)
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
