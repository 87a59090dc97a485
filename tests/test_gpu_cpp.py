"""Build and run the C++ restatement of the reference's own tests
(tests/cpp/test_b200_api.cpp) against the C++ mirror over the C-ABI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_b200_api.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_b200_api")
LIBDIR = os.path.join(ROOT, "paper_2507_16991_b200")
CUDA = "/usr/local/cuda"


def build_cmd():
    return ["g++", "-std=c++20", "-O2", "-ffp-contract=off", SRC, "-o", BIN,
            f"-I{ROOT}/include", f"-I{ROOT}/paper_2507_16991_b200/csrc",
            f"-I{ROOT}/oracle/ref_shim/doctest_shim", f"-I{CUDA}/include",
            f"-L{LIBDIR}", "-lgraphmill_b200", f"-L{CUDA}/lib64", "-lcudart", "-lpthread",
            f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{CUDA}/lib64"]


def test_cpp_mirror_compiles():
    """CPU-side: the header-only mirror and the restated tests compile and link."""
    out = subprocess.run(build_cmd(), capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]


@pytest.mark.gpu
def test_cpp_mirror_runs_reference_cases_on_b200():
    out = subprocess.run(build_cmd(), capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]
    run = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(run.stdout[-2000:], run.stderr[-2000:])
    assert run.returncode == 0, run.stdout[-3000:] + run.stderr[-3000:]
    assert "0 failed" in run.stdout
