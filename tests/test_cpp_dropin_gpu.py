"""The reference-shaped C++ API (include/semlab_b200.hpp) compiles against the C-ABI library and
runs the reference call sequence on the GPU (a C++ caller switching from semlab)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(out):
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "drop_in_example.cpp"), "-o", out,
           "-L", os.path.join(ROOT, "paper_2110_07663_b200"), "-lsemlab_b200",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2110_07663_b200')}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_dropin_compiles(tmp_path):
    _build(str(tmp_path / "dropin"))


@pytest.mark.gpu
def test_cpp_dropin_runs(tmp_path):
    exe = str(tmp_path / "dropin")
    _build(exe)
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.startswith("OK"), p.stdout + p.stderr
