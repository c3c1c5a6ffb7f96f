"""The reference's own doctest unit suites (proj/tests/test_*.cpp, unmodified,
compiled where they lie by `make -C oracle unittests`) run against this
repository's drop-in headers and libsigk.so, with a minimal doctest-compatible
harness (tests/cpp/doctest_shim/doctest.h). tensor_algebra is host-side (runs
without a GPU); the other suites drive the GPU kernels. test_path_io (path CSV
I/O) is out of scope."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "unit_tests_dropin")


def run_suite(suite):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/unit_tests_dropin not built (needs the reference sources at build time)")
    r = subprocess.run([EXE, f"--test-suite={suite}"], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed |" in r.stdout and "test cases: 0 " not in r.stdout


def test_reference_unit_suite_tensor_algebra():
    run_suite("tensor_algebra")


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["kernels", "oracle", "autodiff", "model", "bench"])
def test_reference_unit_suite_on_gpu(suite):
    run_suite(suite)
