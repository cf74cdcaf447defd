"""The C++ host API (include/cftft_b200.hpp) through its test program
tests/cpp/api_test.cpp: validation on CPU, device / host round trips on GPU."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_0810_3203_b200", "lib", "api_test")


def _binary():
    from paper_0810_3203_b200._build import build_api_test, build_library

    build_library()
    return build_api_test()


def test_cpp_api_validation():
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_api_round_trip_on_gpu():
    r = subprocess.run([_binary(), "--gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
