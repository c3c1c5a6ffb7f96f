"""The C++ drop-in API: builds tests/cpp/test_dropin.cpp (reference test cases
restated against include/sigkit/*.hpp) against libsigk.so; runs it on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")
LIBDIR = os.path.join(ROOT, "paper_2501_08455_b200")


def build():
    cmd = ["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), SRC, "-o", BIN,
           "-L" + LIBDIR, "-lsigk", "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return BIN


def test_dropin_headers_compile_and_link():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu():
    r = subprocess.run([build()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
