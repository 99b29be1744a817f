"""Builds and runs the C++ drop-in parity test (tests/cpp/test_dropin.cpp)
against the unmodified reference library. The build step runs everywhere
(g++ only); the run needs a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build():
    lib = os.path.join(ROOT, "paper_1605_00561_b200")
    ref = os.path.join(ROOT, "oracle", "_ref")
    cmd = ["g++", "-std=c++17", "-O2", "-o", BIN, os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
           "-L" + lib, "-lwavelift_b200", "-L" + ref, "-lwavelift_ref",
           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}:{ref}:/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_dropin_compiles():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libwavelift_ref.so")):
        pytest.skip("oracle/_ref not built")
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
