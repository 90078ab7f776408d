"""K2's log1p (csrc/fastmath.cuh) against long-double log1p on the host:
< 1 ulp over 10^7 points covering the feature and softplus ranges.  The same
header compiles for the device; the GPU parity tests check it end to end."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_log1p_fast_under_one_ulp(tmp_path):
    exe = str(tmp_path / "check_log1p")
    subprocess.run(["g++", "-O2", "-I", os.path.join(ROOT, "paper_2012_07145_b200", "csrc"),
                    os.path.join(ROOT, "tools", "check_log1p.cpp"), "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max error 0." in r.stdout
