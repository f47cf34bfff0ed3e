"""Builds tests/cpp/test_adapter.cpp against include/specmc_b200.hpp and the
library, and runs it: on CPU the validation / no-fallback behaviour, on the
GPU (-m gpu) a small model selection through the C++ adapter."""
import subprocess
from pathlib import Path

import pytest

import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def _build(tmp_path):
    exe = tmp_path / "test_adapter"
    lib = _lib.LIB_PATH
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "test_adapter.cpp"),
                    str(lib), f"-Wl,-rpath,{lib.parent}", "-o", str(exe)], check=True)
    return exe


@pytest.mark.skipif(S.device_count() > 0, reason="CPU-only behaviour")
def test_cpp_adapter_cpu(tmp_path):
    r = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_adapter_gpu(tmp_path):
    r = subprocess.run([str(_build(tmp_path)), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
