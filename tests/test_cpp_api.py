"""The C++ drop-in header (include/mrf/mp_cuda.hpp) compiles against the
C-ABI, and on a GPU its reference-signature calls match the C restatement
(tests/cpp/host_api_test.cpp)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA_INC = "/usr/local/cuda/include"
CUDA_LIB = "/usr/local/cuda/lib64"


def _compile(out):
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("no g++")
    lib = os.path.join(ROOT, "paper_1910_10892_b200")
    olib = os.path.join(ROOT, "oracle", "lib")
    cmd = [cxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "oracle"),
           "-I", CUDA_INC, os.path.join(ROOT, "tests", "cpp", "host_api_test.cpp"), "-o", out,
           "-L", lib, "-lmrf_cuda", "-L", olib, "-lmrf_oracle", "-L", CUDA_LIB, "-lcudart",
           f"-Wl,-rpath,{lib}:{olib}:{CUDA_LIB}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


def test_cpp_dropin_header_compiles(tmp_path):
    _compile(str(tmp_path / "host_api_test"))


@pytest.mark.gpu
def test_cpp_dropin_matches_restatement(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = str(tmp_path / "host_api_test")
    _compile(exe)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "OK" in res.stdout
