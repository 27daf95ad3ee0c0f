#!/usr/bin/env python
"""Benchmark: Frank-Wolfe iterations/s of the multi-product newsvendor on B200.

Workload (BASELINE.json configs[1], the config the metric is quoted on):
  newsvendor, d = 10,000 products, S = 100,000 demand scenarios per epoch,
  M = 25 FW iterations per resampling epoch, fp64, seed 42 (instance stream
  (42,0), optimizer stream (42,2): sobench bench.py:40-41, :156-157).
One bench step = one resampling epoch = 1 resample (d*S Philox+Box-Muller
draws, 8 GB) + 25 FW iterations; value = FW iterations/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 shards the SAME problem's products across the N GPUs (strong scaling):
each rank draws and scans only its products (Philox counter offset, no RNG
communication); every FW step exchanges the per-rank LMO argmins inside the
step kernel over NVLink peer memory (CUDA IPC mailboxes; NCCL allgather if IPC
is unavailable) and each epoch's recorded sums once (NCCL allreduce).  See
DESIGN.md section 5.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D, S, M, SEED = 10_000, 100_000, 25, 42
CPU_SAMPLE_D = 1_000  # reference CPU arm: products per bounded sample (cost is linear in d)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the N>1 path with several ranks on one GPU")
    return ap.parse_args()


def dist_setup(n, backend="nccl"):
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dev = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    return rank, world


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


def profiled_traffic():
    """DRAM bytes per k_nv_resample launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_inputs.json")) as fh:
            return json.load(fh).get("k_nv_resample", {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------- CPU reference
def reference_available():
    return os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "sobench"))


def time_reference_epoch(d_sample, threads):
    """One sobench FW epoch (resample + M iterations) at d_sample products, S draws."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_simopt")
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    from sobench import _kernels
    from sobench.backend import make_backend
    from sobench.bench import gen_newsvendor_instance
    from sobench.frank_wolfe import FwConfig, fw_run
    from sobench.sampling import RngStream
    from sobench.tasks import NewsvendorProblem
    _kernels.warmup()
    b = make_backend("parallel", workers=threads)
    task = gen_newsvendor_instance(d_sample, RngStream(SEED, 0))
    prob = NewsvendorProblem(task, b)
    t = time.perf_counter()
    fw_run(prob, FwConfig(1, M, S, RngStream(SEED, 2)), b)
    return time.perf_counter() - t


def time_port_epoch(d_sample):
    """Fallback CPU baseline: the C oracle port (single thread)."""
    from oracle import oracle as orc
    task = orc.gen_newsvendor_instance(d_sample, orc.Stream(SEED, 0))
    t = time.perf_counter()
    orc.fw_run_newsvendor(task, 1, M, S, orc.Stream(SEED, 2))
    return time.perf_counter() - t


def cpu_baseline(steps=1):
    threads = os.cpu_count() or 1
    if reference_available():
        ts = [time_reference_epoch(CPU_SAMPLE_D, threads) for _ in range(steps)]
        kind, cores = "reference", threads
    else:
        ts = [time_port_epoch(CPU_SAMPLE_D) for _ in range(steps)]
        kind, cores = "port", 1
    t = min(ts) if steps == 1 else statistics.mean(ts)
    value = M / (t * D / CPU_SAMPLE_D)
    return {"value": value, "unit": "iterations/s", "cores": cores, "kind": kind,
            "sample": (f"1 FW epoch (resample S={S} + {M} iterations) at d={CPU_SAMPLE_D} products "
                       f"({t:.2f} s), scaled linearly to d={D}; sobench ParallelBackend"
                       if kind == "reference" else
                       f"1 FW epoch at d={CPU_SAMPLE_D} via the C oracle port, scaled to d={D}")}


def run_reference(args, rank):
    if rank != 0:
        return
    ts = []
    for i in range(args.warmup + args.steps):
        if reference_available():
            t = time_reference_epoch(CPU_SAMPLE_D, os.cpu_count() or 1)
        else:
            t = time_port_epoch(CPU_SAMPLE_D)
        if i >= args.warmup:
            ts.append(t * D / CPU_SAMPLE_D)
    per_step = statistics.mean(ts)
    value = M / per_step
    kind = "reference" if reference_available() else "port"
    cores = (os.cpu_count() or 1) if kind == "reference" else 1
    line = {
        "impl": "reference", "metric": "newsvendor Frank-Wolfe iterations/sec (d=10000, S=100000, M=25)",
        "value": value, "unit": "iterations/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "newsvendor C2 (BASELINE.json configs[1])", "d": D, "S": S, "M": M,
                   "seed": SEED},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores, "kind": kind,
                         "sample": f"each step = 1 FW epoch at d={CPU_SAMPLE_D} scaled to d={D}"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- ours
def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist
    import paper_2404_11631_b200 as pkg
    from paper_2404_11631_b200.frank_wolfe import FwConfig, fw_run
    from paper_2404_11631_b200.instances import gen_newsvendor_instance
    from paper_2404_11631_b200.records import TraceBuilder
    from paper_2404_11631_b200.tasks import NewsvendorProblem, make_nv_engine

    from paper_2404_11631_b200.sharding import ShardGroup
    backend = pkg.make_backend("cuda")
    task = gen_newsvendor_instance(D, pkg.RngStream(SEED, 0))
    shard = ShardGroup() if world > 1 else None
    prob = NewsvendorProblem(task, backend, shard=shard)
    epochs = args.warmup + args.steps
    eng = make_nv_engine(prob, M, epochs, backend.chunk_size)  # CUDA-graph epochs
    stream = pkg.RngStream(SEED, 2)
    eng.start()
    for k in range(args.warmup):  # the next epoch's resample overlaps this epoch's steps,
        nxt = S if k + 1 < args.warmup else None  # never across the timed-region boundary
        eng.enqueue_epoch(k, stream, S, next_samples=nxt)
    eng.finish()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record()
        for k in range(args.warmup, epochs):
            nxt = S if k + 1 < epochs else None
            eng.enqueue_epoch(k, stream, S, time_resample=True, next_samples=nxt)
        eng.finish()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # validate the whole run (trace rows, feasibility) outside the timed region
    trace = TraceBuilder()
    for k in range(epochs):
        bad = eng.check_epoch(k, trace)
        if bad:
            raise RuntimeError(f"bench run aborted at step {bad[0]}: {bad[1]}")
    value = args.steps * M / (ms / 1e3)  # one problem, all ranks (strong scaling)
    res_ms = statistics.mean(a.elapsed_time(b) for a, b in eng.resample_events)
    from paper_2404_11631_b200.tasks import nv_geometry
    seg, nbuck = nv_geometry()
    nseg = -(-S // seg)
    d_loc = prob.dev.d
    # the algorithmic bytes of a resample launch are the epoch's fp64
    # demand matrix written once, 8 B per draw (the reference's data model).  This
    # kernel actually writes 4 B keys + 2-byte bucket starts per 4096-draw segment
    # (keyed layout), measured as `traffic`.
    alg_bytes = d_loc * S * 8
    stored_bytes = d_loc * S * 4 + d_loc * nseg * nbuck * 2
    peak, peak_kind = peaks()
    achieved = alg_bytes / (res_ms / 1e3) / 1e9
    traffic = profiled_traffic()  # captured at N=1 (all d products): this rank's share
    if traffic is not None:
        traffic = int(round(traffic * d_loc / D))
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "k_nv_resample", "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "algorithmic_bytes_per_launch": alg_bytes, "stored_bytes_per_launch": stored_bytes,
                "kernel_ms": res_ms, "share_of_step": res_ms / (ms / args.steps),
                "note": ("instruction-bound by design: Philox4x64-10 (37 IMAD/draw) + an fp32 SFU "
                         "Box-Muller key per draw, exact glibc Box-Muller only for the few "
                         "ambiguous draws at query time; kernel_ms is measured while the previous "
                         "epoch's FW steps run concurrently; see profiles/")}
    # the step against SURVEY 8(d)'s per-iteration roof (8 d S (1 + 1/M) bytes: one scan of
    # the epoch's demands per gradient + the amortised write) -- the keyed ECDF reads a
    # window of buckets per product instead of all S demands, so it runs above that roof
    it_roof = peak * 1e9 / (8 * D * S * (1 + 1 / M))
    step_roofline = {"unit": "iterations/s", "data_model_roof": it_roof, "achieved": value,
                     "frac": value / it_roof,
                     "basis": "SURVEY 8(d) C2: 8*d*S*(1+1/M) bytes per FW iteration at hbm peak"}
    launches_per_epoch = 4 * M + 2  # resample, M+1 fused steps, M x (terms, sums, stamp)
    if world > 1 and eng.mailbox is None:
        launches_per_epoch += 2 * M  # LMO pack + apply around each NCCL exchange
    line = {
        "metric": "newsvendor Frank-Wolfe iterations/sec (d=10000, S=100000, M=25)",
        "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "newsvendor C2 (BASELINE.json configs[1])", "d": D, "S": S, "M": M,
                   "seed": SEED, "step": "1 resampling epoch = 1 resample + 25 FW iterations",
                   "l2": "inputs larger than L2 (8 GB demands per epoch)",
                   "parallelism": (f"products sharded x{world}; per-step LMO exchange "
                                   + ("inside the step kernel over NVLink peer memory (CUDA IPC)"
                                      if eng.mailbox is not None else
                                      f"by {args.dist_backend} allgather"))
                   if world > 1 else "single GPU"},
        "roofline": roofline,
        "step_roofline": step_roofline,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_epoch * args.steps,
        "final_objective": trace.build("newsvendor", D, "cuda", 0, SEED, None).final_objective,
    }
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, task, backend, shard)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_e2e(args, task, backend, shard=None):
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
    rec = fw_run(NewsvendorProblem(task, backend, shard=shard), FwConfig(2, M, S, pkg.RngStream(SEED, 2)),
                 backend)  # warm: allocations, layouts, streams
    torch.cuda.synchronize()
    if shard is not None:
        shard.barrier()
    t = time.perf_counter()
    rec = fw_run(NewsvendorProblem(task, backend, shard=shard),
                 FwConfig(steps, M, S, pkg.RngStream(SEED, 2)), backend)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if shard is not None:  # max over ranks
        import torch.distributed as dist
        tt = torch.tensor([dt], dtype=torch.float64,
                          device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    assert rec.iterations.size == steps * M
    h2d = 6 * D * 8 / steps + 4 * 8  # instance once per run (amortised) + the epoch's draw words
    d2h = M * (4 + 8 + 8 + 8) + D * 8 / steps  # per-epoch trace rows + the final iterate (amortised)
    return {"value": steps * M / dt, "unit": "iterations/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "epochs": steps,
            "note": "one fw_run call of `epochs` epochs from host instance arrays (run_cell's call)"}


def main():
    args = parse()
    if args.impl == "reference":
        # host-CPU arm: rank 0 alone times the reference; other ranks exit at once
        run_reference(args, int(os.environ.get("RANK", "0")))
        return
    rank, world = dist_setup(args.gpus, args.dist_backend)
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
