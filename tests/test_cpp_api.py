"""Compiles tests/cpp/test_tsidx_api.cpp against the C++ drop-in API
(include/tsidx/tsidx.hpp) and libtsgpu.so; runs it on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_tsidx_api.cpp")
PKG = os.path.join(ROOT, "paper_2009_00786_b200")


def _compile(tmp_path):
    exe = str(tmp_path / "test_tsidx_api")
    cxx = os.environ.get("CXX", "g++")
    subprocess.run([cxx, "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), SRC, "-o", exe,
                    "-L" + PKG, "-ltsgpu", "-Wl,-rpath," + PKG], check=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    exe = _compile(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK: 0 failures" in out.stdout
