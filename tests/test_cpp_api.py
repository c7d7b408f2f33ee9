"""Compile and run the C++ drop-in API driver (tests/cpp/test_dropin.cpp) against
include/tapt/*.hpp + libtapt_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2509_23043_b200", "lib")
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")


@pytest.fixture(scope="module")
def binary():
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    if not os.path.exists(os.path.join(LIBDIR, "libtapt_b200.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2509_23043_b200", "csrc")], check=True)
    deps = [src] + [os.path.join(ROOT, "include", "tapt", f) for f in os.listdir(os.path.join(ROOT, "include", "tapt"))]
    deps.append(os.path.join(ROOT, "include", "tapt_gpu.h"))
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(os.path.getmtime(d) for d in deps):
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR,
                        "-ltapt_b200", f"-Wl,-rpath,{LIBDIR}", "-o", BIN], check=True)
    return BIN


def test_cpp_dropin_cpu(binary):
    r = subprocess.run([binary, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "cpu ok" in r.stdout


@pytest.mark.gpu
def test_cpp_dropin_gpu(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "gpu ok" in r.stdout
