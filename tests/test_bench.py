"""bench.py's contract: the reference arm (CPU), the self-launching multi-rank run and
the per-task entries (GPU), at the --tiny test sizes."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _line(cmd, timeout):
    out = subprocess.run([sys.executable, BENCH, *cmd], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "sobench")),
                    reason="reference not installed in baseline/_ref")
def test_reference_arm_same_config():
    """--impl reference runs the real sobench fw_run at the config it reports (no
    extrapolation): each step is one full epoch read from the run's own trace."""
    r = _line(["--impl", "reference", "--tiny", "--steps", "2", "--warmup", "1"], 600)
    assert r["impl"] == "reference" and r["config"]["d"] == 2000 and r["config"]["S"] == 5000
    assert r["cpu_baseline"]["kind"] == "reference" and r["value"] > 0
    assert r["e2e"]["h2d_bytes_per_step"] == 0 and r["e2e"]["value"] == r["value"]


@pytest.mark.gpu
def test_bench_two_ranks_self_launch():
    """`bench.py --gpus 2` outside torchrun re-launches itself as two ranks (gloo: both on
    cuda:0 here) and reports n_gpus 2 with the sample-sharded tasks."""
    r = _line(["--gpus", "2", "--dist-backend", "gloo", "--tiny", "--steps", "2", "--warmup", "3",
               "--tasks", "c3,c4,c5", "--no-e2e"], 900)
    assert r["n_gpus"] == 2
    for t in ("c3", "c4", "c5"):
        assert r["per_task"][t]["n_gpus"] == 2 and r["per_task"][t]["value"] > 0, t
    assert 0 < r["per_task"]["c4"]["rows_per_gpu"] < 50_000


@pytest.mark.gpu
def test_bench_one_gpu_all_tasks():
    r = _line(["--tiny", "--steps", "2", "--warmup", "3"], 900)
    assert r["n_gpus"] == 1 and r["value"] > 0 and r["roofline"]["frac"] > 0
    assert r["e2e"]["value"] > 0 and r["cpu_baseline"]["value"] > 0
    for t in ("c1", "c3", "c4", "c5"):
        e = r["per_task"][t]
        assert e["value"] > 0 and e["roofline"]["frac"] > 0, t
        assert "clocks" in e or all("clocks" in v for v in e["variants"]), t
