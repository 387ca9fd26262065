"""The C++ facade (include/subgcache_b200.hpp) compiles against the C ABI here and runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2505_10951_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")


def build(tmp_path):
    exe = str(tmp_path / "facade_test")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"), SRC, "-o", exe,
                    "-L" + LIBDIR, "-lsgc_b200", "-Wl,-rpath," + LIBDIR], check=True)
    return exe


def test_facade_compiles(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_facade_runs_on_gpu(tmp_path):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade ok" in out.stdout
