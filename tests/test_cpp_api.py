"""Runs the C++ drop-in check (tests/cpp/test_api.cpp: reference test bodies over include/moses_gpu.hpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_api_reference_cases():
    from paper_2201_05752_b200 import build as b

    b.build()
    exe = os.path.join(ROOT, "paper_2201_05752_b200", "_build", "test_api")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: 0 failure(s)" in r.stdout


def test_cpp_api_builds():
    from paper_2201_05752_b200 import build as b

    b.build()
    assert os.path.exists(os.path.join(ROOT, "paper_2201_05752_b200", "_build", "test_api"))
