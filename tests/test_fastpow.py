"""Accuracy of the device pow replacement (csrc/nlg_math.cuh), compiled for
the host with nvcc and checked against libm pow (no GPU needed)."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fast_pow_accuracy(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = tmp_path / "fastpow_check"
    subprocess.run([nvcc, "-O2", "-Wno-deprecated-gpu-targets", "-o", str(exe),
                    os.path.join(ROOT, "tests", "native", "fastpow_check.cu")], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, f"max relative error {out.stdout.strip()} exceeds 2e-14"
