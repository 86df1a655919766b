"""The C++ mirror (include/morprec_gpu.hpp) driving the GPU path end to end."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_mirror_runs_on_gpu(mpg, tmp_path):
    exe = tmp_path / "cpp_api_demo"
    libdir = os.path.join(ROOT, "paper_2003_12759_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "cpp_api_demo.cpp"), "-L", libdir, "-lmpg",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
