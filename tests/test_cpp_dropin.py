"""The C++ drop-in API: builds tests/cpp/*.cpp (reference test cases restated
against include/sigkit/*.hpp) against libsigk.so; runs them on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2501_08455_b200")
CASES = ["test_dropin", "test_model_dropin"]


def build(name):
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    exe = os.path.join(ROOT, "tests", "cpp", name)
    cmd = ["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", exe,
           "-L" + LIBDIR, "-lsigk", "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


@pytest.mark.parametrize("name", CASES)
def test_dropin_headers_compile_and_link(name):
    assert os.path.exists(build(name))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_dropin_reference_cases_on_gpu(name):
    r = subprocess.run([build(name)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_dropin_host_dispatch_cases():
    # test_kernels.cpp:299-315 (dispatch, SIGKIT_ACCELERATED): host logic, no GPU needed
    r = subprocess.run([build("test_dropin"), "--host-only"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
