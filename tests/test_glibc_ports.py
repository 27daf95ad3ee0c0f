"""Host check of the device libm ports (csrc/glibc_math.cuh) against this machine's glibc:
the same header the GPU compiles with -fmad=false, built here with -ffp-contract=off."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_erf_port_bitwise_vs_host_glibc(tmp_path):
    """glibc_erf (a port of libm.so.6 `erf`, used by the recorded newsvendor objective,
    _kernels.py:219-220) equals the host erf bit for bit on 2e6 inputs over every region."""
    exe = str(tmp_path / "erf_check")
    cc = subprocess.run(["gcc", "-O2", "-ffp-contract=off",
                         "-I", os.path.join(ROOT, "paper_2404_11631_b200", "csrc"),
                         os.path.join(ROOT, "tests", "native", "erf_check.c"), "-lm", "-o", exe],
                        capture_output=True, text=True)
    if cc.returncode != 0:
        pytest.skip(f"no host C compiler: {cc.stderr[:200]}")
    run = subprocess.run([exe, "2000000"], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0 and run.stdout.strip() == "0", (run.stdout, run.stderr[:500])
