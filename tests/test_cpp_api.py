"""Runs the C++ parity test of the reference-signature API
(include/stitch_b200.hpp, tests/cpp/test_pipeline.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_pipeline")


def test_cpp_binary_builds_or_exists():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_api_parity_with_oracle():
    # incremental: rebuilt whenever the headers changed
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout
