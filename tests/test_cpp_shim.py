"""The C++ mirror (include/embcomm_gpu.hpp) compiles, links against
libembcomm_gpu.so and passes reference-test cases: host cases on CPU,
simulator cases on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2411_01611_b200")


@pytest.fixture(scope="module")
def shim_bin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("shim") / "shim_test")
    cuda_inc = "/usr/local/cuda/include"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", cuda_inc,
                    os.path.join(ROOT, "tests", "cpp", "shim_test.cpp"), "-L", LIBDIR, "-lembcomm_gpu",
                    f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


def test_cpp_shim_host_cases(shim_bin):
    r = subprocess.run([shim_bin], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_shim_gpu_cases(shim_bin):
    r = subprocess.run([shim_bin, "--gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
